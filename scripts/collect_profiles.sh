#!/bin/bash
# Copies the evidence of a GPU job (gpurun_out/<tag>_*) into profiles/ as text summaries (tracked), and refreshes
# profiles/roofline_traffic.json -- the per-workload ncu counters bench.py reads.   scripts/collect_profiles.sh r02
tag=${1:-r02}
cd "$(dirname "$0")/.."
declare -A COST=( [c1_tiny]=10 [c2_planted]=12 [c3_long]=9 [c4_many]=7 [c5_deep]=20 )
for c in c1_tiny c2_planted c3_long c4_many c5_deep; do
  [ -f gpurun_out/${tag}_launches_$c.csv ] || continue
  python scripts/ncu_tables.py launches gpurun_out/${tag}_launches_$c.csv > profiles/${tag}_launches_$c.txt
  mc=$(python -c "from paper_2402_12373_b200 import workloads as W; print(W.CONFIGS['$c']['max_cost'])")
  python scripts/ncu_tables.py traffic gpurun_out/${tag}_launches_$c.csv $c mueller $mc profiles/roofline_traffic.json > /dev/null
  [ -f gpurun_out/${tag}_full_${c}_raw.csv ] && python scripts/ncu_tables.py raw gpurun_out/${tag}_full_${c}_raw.csv > profiles/${tag}_full_${c}_summary.txt
  [ -f gpurun_out/${tag}_full_${c}_source.csv.gz ] && python scripts/ncu_source_hot.py gpurun_out/${tag}_full_${c}_source.csv.gz -1 24 > profiles/${tag}_full_${c}_hot_sass.txt 2>/dev/null
  [ -f gpurun_out/${tag}_bench_$c.json ] && cp gpurun_out/${tag}_bench_$c.json profiles/${tag}_bench_$c.json
done
for f in block_sweep.txt deep_runs.txt; do [ -f gpurun_out/${tag}_$f ] && cut -c1-700 gpurun_out/${tag}_$f > profiles/${tag}_$f; done
[ -f gpurun_out/${tag}_experiments.json ] && python - <<PY
import json
d = json.load(open("gpurun_out/${tag}_experiments.json"))
json.dump({"ruc": {k: d["ruc"][k] for k in ("seeds", "summary", "runs", "wall_s")}, "skipped": len(d["ruc"]["skipped"]),
           "masking_sweep": d["masking_sweep"]}, open("profiles/${tag}_experiments.json", "w"), indent=1)
PY
for f in gpurun_out/${tag}_sanitize_*.log; do
  [ -f "$f" ] || continue
  { echo "# $(basename $f)"; grep -E "COMPUTE-SANITIZER|SUMMARY|^exit|smoke ok|^rowsplit|^budget|^halfwidth|^traces |Race reported|and (Read|Write) access" "$f" | cut -c1-220 | sort | uniq -c | sort -rn | head -14; } 
done > profiles/${tag}_sanitizer.txt
scripts/sass_excerpt.sh paper_2402_12373_b200/csrc/build/screen_w1.o '_Z8k_screenILi1ELi3ELb0EEv12ScreenParams' > profiles/${tag}_sass_k_screen_w1_nh.txt
scripts/sass_excerpt.sh paper_2402_12373_b200/csrc/build/screen_w1.o '_Z17k_materialize_notILi3ELb0ELb1EEv17MaterializeParams12ScreenParams' > profiles/${tag}_sass_k_materialize_not_nh.txt
scripts/sass_excerpt.sh paper_2402_12373_b200/csrc/build/screen_w1.o '_Z17k_materialize_notILi3ELb0ELb0EEv17MaterializeParams12ScreenParams' > profiles/${tag}_sass_k_materialize_not_nh_evalonly.txt
scripts/sass_excerpt.sh paper_2402_12373_b200/csrc/build/screen_w1p.o 'k_screenILi1ELi3ELb1EE' > profiles/${tag}_sass_k_screen_w1_halfwidth.txt
ls -la profiles | tail -40
