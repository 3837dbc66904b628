#!/bin/bash
# Evidence run of round 2 on the GPU box (under gpurun): per-config bench lines, ncu launch lists and full captures
# (scripts/gpu_profile_configs.sh), phase-B block-size sweep, deep runs under both fingerprints, the RUC experiment with
# NH beside MuellerHash.  Everything lands in gpurun_out/ (summaries are copied to profiles/ by hand).
tag=${1:-r02}
for b in 2 4 8 16 32 64; do LTL_CORE_OPTIONS=order_block_bytes=$((b<<20)) timeout 300 python bench.py --config c2_planted --configs none --steps 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('c2 phase-B block MB $b:', round(d['value']/1e6,1), 'M cand/s', round(d['ms_per_step'],2), 'ms/step; materialize ms per 3 steps', d['roofline']['kernel_ms_by_class']['materialize'])"; done > gpurun_out/${tag}_block_sweep.txt 2>&1
cat gpurun_out/${tag}_block_sweep.txt
bash scripts/gpu_profile_configs.sh $tag c1_tiny c2_planted c3_long c4_many c5_deep 2>&1 | grep -v "^$" | cut -c1-400 | tail -60
for hsh in mueller mueller_blocked; do for c in c2_planted c5_deep c3_long; do
  timeout 600 python scripts/profile_target.py --config $c --unsolvable --max-cost 20 --hash $hsh --repeat 2 2>&1 | grep -E "^run|^\[\(" | cut -c1-600 | sed "s/^/deep $c $hsh: /"
done; done > gpurun_out/${tag}_deep_runs.txt 2>&1
cat gpurun_out/${tag}_deep_runs.txt | cut -c1-300
timeout 900 python scripts/run_experiments.py --seeds 10 --hashes mueller,nh,mueller_blocked,fkp --out gpurun_out/${tag}_experiments.json > /dev/null 2>&1
python -c "
import json; d=json.load(open('gpurun_out/${tag}_experiments.json')); print(json.dumps(d['ruc']['summary'])); print(d['ruc']['runs'], d['ruc']['wall_s'])"
