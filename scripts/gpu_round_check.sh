set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/tests_all.log
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3.jsonl 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --steps 3 --warmup 3 --vslabs 2 --halo peer --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_v2peer.jsonl 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --vslabs 4 --halo peer --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_v4peer.jsonl 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --vslabs 2 --halo copy --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_c3_v2copy.jsonl 2>&1
tail -3 gpurun_out/tests_all.log
