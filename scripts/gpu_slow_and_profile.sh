#!/bin/bash
# full-size parity tests (configs[1], configs[2]) + launch list and ncu capture of the persistent cycle kernel (C3)
timeout 1500 python -m pytest tests -m "gpu and slow" -x -q > gpurun_out/gpu_slow.log 2>&1; echo slow=$?
B="python bench.py --workload C3 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --engine persistent"
$B > gpurun_out/plain_c3_persistent.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_persistent.csv $B > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_persistent" -c 1 -o gpurun_out/prof_c3_persistent $B > gpurun_out/ncu_p.log 2>&1
echo done
