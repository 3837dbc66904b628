#!/bin/bash
# Final evidence run after the gated store: the full GPU suite, smoke(), the default bench line and the reference arm, the
# ncu launch list + full capture of config 2 (the only shape whose launches changed), deep runs of three shapes (gate on)
# and config 2's with the gate off.
tag=${1:-r02h}
timeout 1900 python -m pytest tests -m gpu -x -q --timeout 400 2>&1 | tail -6 > gpurun_out/${tag}_gputests.log; cat gpurun_out/${tag}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/${tag}_bench_default.json 2> gpurun_out/${tag}_bench_default.err; tail -c 300 gpurun_out/${tag}_bench_default.json; echo
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_reference.json 2> /dev/null; tail -c 400 gpurun_out/${tag}_bench_reference.json; echo
bash scripts/gpu_profile_configs.sh $tag c2_planted 2>&1 | grep -E "^==|bench:|total" | cut -c1-200 | tail -30
for c in c2_planted c5_deep c3_long; do
  timeout 600 python scripts/profile_target.py --config $c --unsolvable --max-cost 20 --hash mueller --repeat 2 2>&1 | grep -E "^run|^\[\(" | cut -c1-600 | sed "s/^/deep $c mueller: /"
done > gpurun_out/${tag}_deep_runs.txt 2>&1
LTL_CORE_OPTIONS=gate_store=0 timeout 600 python scripts/profile_target.py --config c2_planted --unsolvable --max-cost 20 --hash mueller --repeat 2 2>&1 | grep -E "^run|^\[\(" | cut -c1-600 | sed "s/^/deep c2_planted mueller gate_store=0: /" >> gpurun_out/${tag}_deep_runs.txt
cat gpurun_out/${tag}_deep_runs.txt | cut -c1-300
