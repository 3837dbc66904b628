#!/bin/bash
# scripts/build_variants.sh "name -DX=.. -DY=.." ...   builds core.o once, every W=1 variant object in parallel, links each
# into paper_2402_12373_b200/csrc/variants/libltlcore_<name>.so (needs a complete regular build for the W >= 2 objects)
cd "$(dirname "$0")/../paper_2402_12373_b200/csrc" || exit 1
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden"
mkdir -p variants
nvcc $F -c core.cu -o build/core.o &
names=()
for v in "$@"; do
  read -r n defs <<< "$v"
  names+=("$n")
  (nvcc $F $defs -DLTL_W=1 -c screen_inst.cu -o variants/screen_w1_$n.o 2>&1 | grep -iE "error" ) &
done
wait
for n in "${names[@]}"; do
  objs="build/core.o build/traces.o build/screen_w1p.o variants/screen_w1_$n.o"
  for w in $(seq 2 16); do objs="$objs build/screen_w$w.o"; done
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o variants/libltlcore_$n.so $objs
  echo -n "$n: "; cuobjdump -res-usage variants/screen_w1_$n.o | grep -A1 "k_materialize" | grep -o "REG:[0-9]* STACK:[0-9]*" | tr '\n' ' '; echo
done
