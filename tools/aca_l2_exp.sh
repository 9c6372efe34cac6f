#!/usr/bin/env bash
# ACA working-set experiments (config 3): chain durations against batch size,
# L2 cache-policy variants, persistent-grid caps.  Output: gpurun_out/aca_l2_exp.log
out=gpurun_out/aca_l2_exp.log
: > $out
for B in 8 16 32 64; do
  echo "== profile B=$B" >> $out
  HK_ACA_PROFILE=gpurun_out/acaprof_$B.txt python tools/host_profile.py $B 2>&1 | tail -2 >> $out
done
for v in "" variants/lib_uvel.so variants/lib_srccs.so variants/lib_both.so; do
  echo "== variant '$v'" >> $out
  HK_LIB_PATH=$v python tools/host_profile.py 64 2>&1 | tail -3 >> $out
done
for g in "128,256,512,1024" "64,128,256,512" "96,192,384,768" "128,128,256,512" "64,256,512,1024" "128,256,256,256" "128,192,256,384"; do
  echo "== grid $g" >> $out
  HK_ACA_GRID=$g python tools/host_profile.py 64 2>&1 | tail -2 >> $out
done
echo "== base again" >> $out
python tools/host_profile.py 64 2>&1 | tail -3 >> $out
