#!/bin/bash
# Per-config evidence run on the GPU box (under gpurun): for each BASELINE shape a bench line, the ncu launch list
# (time, warp instructions, DRAM bytes per launch) and one `--set full` capture of the largest k_screen launch.
#   scripts/gpu_profile_configs.sh <tag> [config ...]
# Outputs: gpurun_out/<tag>_bench_<cfg>.json, <tag>_launches_<cfg>.csv, <tag>_full_<cfg>.ncu-rep
tag=${1:-r02}; shift
cfgs=${@:-"c3_long c4_many c5_deep"}
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum
for c in $cfgs; do
  extra=""
  echo "== $c bench"; date
  timeout 900 python bench.py --config $c $extra --steps 3 --warmup 3 > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
  tail -c 600 gpurun_out/${tag}_bench_$c.json
  echo "== $c launches"; date
  timeout 1500 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${tag}_launches_$c.csv \
      python scripts/profile_target.py --config $c $extra > gpurun_out/${tag}_launches_$c.log 2>&1
  tail -3 gpurun_out/${tag}_launches_$c.log
  echo "== $c full"; date
  # the largest k_screen launches are the last ones of the search
  n=$(grep -c k_screen gpurun_out/${tag}_launches_$c.csv)
  n=$((n / 6))
  skip=$((n > 3 ? n - 3 : 0))
  # reports stay in /tmp on the box (gpurun_out is capped at 64 MiB): the raw and source pages come back as CSV
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_screen -s $skip -c 3 -f -o /tmp/${tag}_full_$c \
      python scripts/profile_target.py --config $c $extra > gpurun_out/${tag}_full_$c.log 2>&1
  tail -2 gpurun_out/${tag}_full_$c.log
  ncu -i /tmp/${tag}_full_$c.ncu-rep --page raw --csv > gpurun_out/${tag}_full_${c}_raw.csv 2>/dev/null
  ncu -i /tmp/${tag}_full_$c.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/${tag}_full_${c}_source.csv.gz
  sz=$(stat -c %s /tmp/${tag}_full_$c.ncu-rep 2>/dev/null || echo 0)
  [ "$sz" -gt 0 ] && [ "$sz" -lt 12000000 ] && cp /tmp/${tag}_full_$c.ncu-rep gpurun_out/
  du -sh gpurun_out
done
date
