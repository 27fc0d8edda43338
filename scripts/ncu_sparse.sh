#!/bin/bash
# one mid-run fire + treat of the stepped wheel engine on a thin-front workload (C4) and C2, full sections + source
for W in C4 C2; do
B="python bench.py --workload $W --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --engine wheel_stepped"
$B > gpurun_out/plain_${W}_stepped.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_wheel_fire|k_wheel_treat" -s 1200 -c 2 -o gpurun_out/prof_${W}_stepped $B > gpurun_out/ncu_${W}.log 2>&1
done
echo done
