#!/usr/bin/env bash
for d in "$@"; do
  line=$(HK_ACA_DELAY=$d python tools/host_profile.py 64 2>&1 | tail -2 | sed "s/.*'lowrank': \([0-9.]*\),.*/\1/" | tr '\n' ' ')
  echo "delay $d: $line"
done
