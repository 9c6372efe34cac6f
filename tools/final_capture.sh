#!/usr/bin/env bash
# Round-end capture: GPU suite, bench line, reference line, ncu launch list of a short bench,
# ncu --set full of the ACA class launches (config 3, 64 fronts).  Outputs in gpurun_out/.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/f_gputest.log 2>&1; tail -2 gpurun_out/f_gputest.log
python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_reference.json 2> gpurun_out/f_reference.err; echo "ref rc=$?"
SHORT="python bench.py --steps 2 --warmup 3 --no-cfg12 --no-cfg4 --no-cfg0 --level-fronts 0 --no-e2e --no-cpu-baseline"
$SHORT > gpurun_out/f_short.json 2> gpurun_out/f_short.err &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv $SHORT > gpurun_out/f_ncu_launch.log 2>&1
python tools/host_profile.py 64 > gpurun_out/f_plain64.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:aca_kernel --launch-skip 8 --launch-count 4 -o gpurun_out/aca_r02b python tools/host_profile.py 64 > gpurun_out/f_ncu_aca.log 2>&1
tail -1 gpurun_out/f_ncu_aca.log
