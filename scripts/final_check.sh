#!/bin/bash
# What the driver runs at round end, from the committed state: smoke(), the default bench line (timed), its key fields.
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
SECONDS=0
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
echo "bench.py took ${SECONDS}s, exit $?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/final_bench.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(d["value"] / 1e6, d["ms_per_step"], d["e2e"]["value"] / 1e6, d["gpu_launches"], d["clocks"])
print(r["bound"], r["frac"], r["traffic"], r["profile_build_matches"], r["materialize"].get("dram"), r["materialize"]["frac"])
for k, v in d["configs"].items():
    rr = v["roofline"]
    print(k, v["ms_per_step"], rr["bound"], round(rr["frac"], 3), rr.get("profile_build_matches"), v["clocks"])
PY
