#!/bin/bash
# default bench line + launch list + one ncu --set full capture of the timed cycle kernel (C3, wheel)
python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
for W in C2 C4 C3s; do python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$W.log 2>&1; done
B="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
$B > gpurun_out/plain_default.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv $B > gpurun_out/ncu_d1.log 2>&1
# skip the warm-up solve's cycle kernel, capture the timed one
ncu --set full --clock-control none --import-source on -k regex:"k_wheel_persistent" -s 1 -c 1 -o gpurun_out/prof_default $B > gpurun_out/ncu_d2.log 2>&1
echo done
