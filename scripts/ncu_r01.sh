#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run first, then ncu on the same command.
set -x
B="python bench.py --workload C3s --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
$B --engine stepped > gpurun_out/plain_stepped.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_stepped.csv $B --engine stepped > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_treat" -s 400 -c 4 -o gpurun_out/prof_stepped $B --engine stepped > gpurun_out/ncu2.log 2>&1
$B --engine persistent > gpurun_out/plain_persistent.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_persistent" -c 1 -o gpurun_out/prof_persistent $B --engine persistent > gpurun_out/ncu3.log 2>&1
echo done
