timeout 900 python -m pytest tests -m "gpu" -x -q 2>&1 | tail -2
VARIANTS="prev" WS="C3 C2 C3s C4" bash scripts/ab_bench.sh
for v in base prev; do
  if [ $v = base ]; then lib=paper_1511_06441_b200/libwcsp.so; else lib=paper_1511_06441_b200/libwcsp_$v.so; fi
  for k in 2 4; do echo "== vslabs $k $v $(WCSP_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 3 --vslabs $k --halo peer --no-cpu-baseline --e2e-steps 0 2>/dev/null | grep '^{' | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"; done
done
