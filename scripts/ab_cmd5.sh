L=paper_1511_06441_b200
timeout 700 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
VARIANTS="nofpf prev fi4" WS="C3 C2" bash scripts/ab_quick.sh
for v in base nopr; do
  if [ $v = base ]; then lib=$L/libwcsp.so; else lib=$L/libwcsp_$v.so; fi
  for k in 2 4; do echo "== vslabs $k $v $(WCSP_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 3 --vslabs $k --halo peer --no-cpu-baseline --e2e-steps 0 2>/dev/null | grep '^{' | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"])')"; done
done
