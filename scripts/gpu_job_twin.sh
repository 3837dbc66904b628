#!/bin/bash
# A/B of the evaluate-only twin of the fused phase B (launch bounds x unroll) on the bench workload + a fused-NOT test pass
tag=${1:-twin}
timeout 900 python -m pytest tests/test_gpu_core.py tests/test_gpu_fullsize.py tests/test_gpu_halfwidth.py -x -q -m gpu --timeout 300 -k "fused or full or half or golden" 2>&1 | tail -3 | cut -c1-300
AB_ARGS="--config c2_planted --configs none --steps 5 --warmup 3" bash scripts/ab_bench.sh $tag base e2u16 e3u16 e4u8 e4u4 base:gate_store=0 2>&1 | cut -c1-200
bash scripts/gpu_job_matnot.sh ${tag}_matnot 2>&1 | tail -3
