#!/bin/bash
# quick perf set: C3 and C2 for the given engines (no cpu baseline)
for e in ${ENGINES:-wheel persistent}; do
  for w in ${WORKLOADS:-C3 C2}; do
    timeout 300 python bench.py --workload $w --engine $e --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_${w}_$e.log 2>&1
    echo "$w $e rc=$?"
  done
done
