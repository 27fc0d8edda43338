#!/bin/bash
# one mid-run fire + treat of the stepped wheel engine on C3 (full sections + source), plus the launch list
B="python bench.py --workload C3 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --engine wheel_stepped"
$B > gpurun_out/plain_C3_stepped.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_wheel_fire|k_wheel_treat" -s 900 -c 2 -o gpurun_out/prof_C3_stepped $B > gpurun_out/ncu_C3s.log 2>&1
echo done
