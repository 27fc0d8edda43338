#!/bin/bash
# ncu --set full on one mid-run sweep and treat launch of the stepped engine (C3 256^3)
B="python bench.py --workload C3 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --engine stepped"
$B > gpurun_out/plain_c3_stepped.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_sweep|k_treat" -s 800 -c 2 -o gpurun_out/prof_c3_stepped $B > gpurun_out/ncu_c3.log 2>&1
echo done
