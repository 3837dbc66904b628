#!/bin/bash
# ncu --set full capture of the evaluate-only twin of the fused phase B on config 2 (the 5th k_materialize_not launch of a
# search: cost level 11 finds its gate closed)
tag=${1:-evalonly}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_materialize_not -s 4 -c 1 -f -o /tmp/${tag}_full \
    python scripts/profile_target.py --config c2_planted > gpurun_out/${tag}_full.log 2>&1
tail -2 gpurun_out/${tag}_full.log
ncu -i /tmp/${tag}_full.ncu-rep --page raw --csv > gpurun_out/${tag}_full_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_full.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/${tag}_full_source.csv.gz
