#!/bin/bash
# v14b: per-build fire chunk (12 events per lane in the 4-block build; 6 in dense cycles of the 3-block build)
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_v14b.log 2>&1; echo tests=$?
timeout 300 python bench.py > gpurun_out/bench_c3_v14b.log 2>&1; echo bench=$?
for W in C2 C4 C3s; do for rep in 1 2; do timeout 200 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | grep '^{' >> gpurun_out/bench_${W}_v14b.jsonl; done; done
echo done
