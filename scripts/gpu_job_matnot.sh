#!/bin/bash
# ncu --set full capture of the fused phase-B launches of config 2 (the last one finds its gate closed: eval-only)
tag=${1:-matnot}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_materialize_not -c 3 -f -o /tmp/${tag}_full \
    python scripts/profile_target.py --config c2_planted > gpurun_out/${tag}_full.log 2>&1
tail -2 gpurun_out/${tag}_full.log
ncu -i /tmp/${tag}_full.ncu-rep --page raw --csv > gpurun_out/${tag}_full_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_full.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/${tag}_full_source.csv.gz
ls -la gpurun_out | tail -4
