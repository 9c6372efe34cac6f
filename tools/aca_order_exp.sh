#!/usr/bin/env bash
# each argument: "ORDER;PRIO;DELAY" (empty fields = default)
for a in "$@"; do
  IFS=';' read -r o p d <<< "$a"
  line=$(env ${o:+HK_ACA_ORDER=$o} ${p:+HK_ACA_PRIO=$p} ${d:+HK_ACA_DELAY=$d} python tools/host_profile.py ${B:-64} 2>&1 | tail -2 | sed "s/.*'lowrank': \([0-9.]*\),.*/\1/" | tr '\n' ' ')
  echo "order=$o prio=$p delay=$d: $line"
done
