timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/tests12.log
timeout 300 python bench.py > gpurun_out/bench12.jsonl 2> gpurun_out/bench12.err
timeout 1500 python bench.py --workload C5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_C5_12.jsonl 2> gpurun_out/bench_C5_12.err
