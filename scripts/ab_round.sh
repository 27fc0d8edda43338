echo "== peer tests"; timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "peer or reuse" 2>&1 | tail -1
timeout 250 python scripts/peer_det.py
for v in 2 4; do timeout 300 python bench.py --steps 3 --warmup 3 --vslabs $v --halo peer --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('vslabs', $v, d['ms_per_step'])"; done
