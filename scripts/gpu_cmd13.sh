timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "both_cycle or peer or slab" 2>&1 | tail -3
for k in 2 4; do echo "== vslabs $k peer $(timeout 300 python bench.py --steps 3 --warmup 3 --vslabs $k --halo peer --no-cpu-baseline --e2e-steps 0 2>/dev/null | grep '^{' | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["solve"]["F1"], d["solve"]["edge_updates"])')"; done
VARIANTS="fl2k fl1k" WS="C3" bash scripts/ab_bench.sh
