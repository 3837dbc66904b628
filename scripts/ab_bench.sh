#!/bin/bash
# A/B of variant libraries on the bench workload: scripts/ab_bench.sh <tag> <variant>...   ("base" = the regular build;
# a trailing ":opt=val,..." sets LTL_CORE_OPTIONS for that run).  One JSON line per variant in gpurun_out/ab_<tag>_<variant>.json.
tag=$1; shift
for spec in "$@"; do
  v=${spec%%:*}; opts=""; [[ "$spec" == *:* ]] && opts=${spec#*:}
  lib=""; [ "$v" != base ] && lib=$PWD/paper_2402_12373_b200/csrc/variants/libltlcore_$v.so
  out=gpurun_out/ab_${tag}_${spec//[:=,]/_}.json
  LTL_CORE_LIB=$lib LTL_CORE_OPTIONS=$opts python bench.py --no-cpu-baseline ${AB_ARGS} > $out 2> gpurun_out/ab_${tag}.err
  python - "$spec" $out <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
k = d["roofline"]["kernel_ms_by_class"]
print(f"{sys.argv[1]:24s} {d['value']/1e6:7.1f} Mc/s {d['ms_per_step']:7.2f} ms  e2e {d['e2e']['value']/1e6:7.1f}  screen {k['screen']/d['steps']:6.2f} mat {k['materialize']/d['steps']:6.2f} ms/step")
PY
done
