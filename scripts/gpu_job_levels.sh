#!/bin/bash
# Iteration job for the device-resident levels / small-pass kernels: tests, per-phase traces, bench lines, a short soak.
tag=${1:-lv}
timeout 900 python -m pytest tests/test_gpu_core.py tests/test_gpu_fullsize.py -x -q -m gpu --timeout 300 2>&1 | tail -3 | cut -c1-300 > gpurun_out/${tag}_tests.log; cat gpurun_out/${tag}_tests.log
for c in c1_tiny c2_planted c5_deep; do LTL_LEVELS_TRACE=1 python scripts/c1_probe.py $c 3 2>&1 | grep -E "^levels|per search" | cut -c1-300 | tail -8; done
for c in c1_tiny c5_deep c2_planted; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  python - <<PY | cut -c1-900
import json
d = json.loads(open("gpurun_out/${tag}_bench_$c.json").read().strip().splitlines()[-1])
print("$c", round(d["ms_per_step"], 4), round(d["e2e"]["ms_per_step"], 4), d.get("levels"), d["roofline"].get("kernel_ms_by_class"), d["gpu_launches"])
PY
  tail -3 gpurun_out/${tag}_bench_$c.err | cut -c1-300
done
timeout 300 python scripts/soak.py --seconds ${2:-150} --seed 12 2>&1 | tail -2 | cut -c1-300
