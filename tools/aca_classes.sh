#!/usr/bin/env bash
# per-class ACA kernel times (ncu launch list, serialised) for one config-3 build:
#   tools/aca_classes.sh <tag> [env...]
tag=$1; shift
env "$@" ncu --metrics gpu__time_duration.sum --clock-control none -k regex:aca_kernel \
  --launch-skip 8 --launch-count 4 --csv python tools/host_profile.py 64 2>/dev/null \
  | grep aca_kernel | awk -F'","' -v t="$tag" '{print t, $5, $NF}' | sed 's/"//g'
