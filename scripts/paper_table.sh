#!/bin/bash
# §6 protocol replica: our solve time on the four cubes, binding M and M = infinity,
# with the oracle's time on the host (bench cpu_baseline leg) beside it.
for s in 50 75 100 125; do
  for m in "" "-inf"; do
    timeout 600 python bench.py --workload P6-$s$m --steps 5 --warmup 3 --e2e-steps 0 --ref-seconds 60 > gpurun_out/p6_$s$m.log 2>&1
    echo "P6-$s$m rc=$?"
  done
done
