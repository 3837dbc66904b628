#!/bin/bash
# re-run one soak case (seed $1, case $2) over the hand-over options of the device-resident levels
seed=${1:-12}; n=${2:-84}
for opts in "levels_ctas=8,levels_max_work=16777216" "levels_ctas=1,levels_max_work=16777216" "levels_ctas=4,levels_max_work=262144" "levels_ctas=2,levels_max_work=16384"; do
  echo "== $opts"
  for rep in 1 2 3; do
  SOAK_ONLY=$n SOAK_LEVELS_OPTS=$opts LTL_LEVELS_TRACE=1 timeout 300 python scripts/soak.py --seconds 100 --seed $seed 2>&1 | grep -E "MISMATCH|got|soak ok|levels:" | cut -c1-330 | tail -12
  done
done
