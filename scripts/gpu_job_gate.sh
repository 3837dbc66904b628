#!/bin/bash
# Verification job of the gated store: the GPU tests with the gate forced on for every core, an A/B of the
# bench workload (gate_store=0 / 1), the deep unsolvable run both ways, a short soak.
tag=${1:-gate}
export LTL_CORE_OPTIONS=gate_store=1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 400 2>&1 | tail -4 | cut -c1-300 > gpurun_out/${tag}_tests.log; cat gpurun_out/${tag}_tests.log
for g in 0 1; do
  export LTL_CORE_OPTIONS=gate_store=$g
  timeout 600 python bench.py --config c2_planted --steps 5 --warmup 3 > gpurun_out/${tag}_bench_c2_g$g.json 2> gpurun_out/${tag}_bench_c2_g$g.err
  python - <<PY | cut -c1-700
import json
d = json.loads(open("gpurun_out/${tag}_bench_c2_g$g.json").read().strip().splitlines()[-1])
print("gate=$g", round(d["ms_per_step"], 3), round(d["e2e"]["ms_per_step"], 3), round(d["value"] / 1e6, 1), d["formula"], d["candidates_per_step"], d["unique_cs_per_step"], d["roofline"].get("kernel_ms_by_class"), d["gpu_launches"])
PY
  tail -2 gpurun_out/${tag}_bench_c2_g$g.err | cut -c1-300
  timeout 600 python scripts/profile_target.py --config c2_planted --unsolvable --max-cost 20 --budget-gb 150 2>&1 | tail -3 | cut -c1-400
done
export LTL_CORE_OPTIONS=gate_store=1
timeout 400 python scripts/soak.py --seconds ${2:-200} --seed 31 2>&1 | tail -2 | cut -c1-300
