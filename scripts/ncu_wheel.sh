#!/bin/bash
# wheel engine: launch list (stepped) + full capture of one mid-run fire/treat (stepped) and of the persistent kernel (C3)
W=${W:-C3}
B="python bench.py --workload $W --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
$B --engine wheel_stepped > gpurun_out/plain_wheel_stepped.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_wheel_stepped.csv $B --engine wheel_stepped > gpurun_out/ncu_w1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_wheel_fire|k_wheel_treat" -s 800 -c 2 -o gpurun_out/prof_wheel_stepped $B --engine wheel_stepped > gpurun_out/ncu_w2.log 2>&1
$B --engine wheel > gpurun_out/plain_wheel.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_wheel_persistent" -c 1 -o gpurun_out/prof_wheel $B --engine wheel > gpurun_out/ncu_w3.log 2>&1
echo done
