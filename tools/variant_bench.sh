#!/usr/bin/env bash
# A/B of variant builds of the library on the config-3 build (tools/host_profile.py):
#   tools/variant_bench.sh <fronts> <rounds> lib1.so lib2.so ...   ("base" = the in-tree library)
# prints, per variant and round, the GPU-timed low-rank build / leaf / schur times of the last iteration
B=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for v in "$@"; do
    if [ "$v" = base ]; then p=""; else p=$v; fi
    line=$(HK_LIB_PATH=$p python tools/host_profile.py $B 2>&1 | tail -1 | sed 's/.*gpu t=//')
    echo "$v round $r: $line"
  done
done
