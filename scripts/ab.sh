#!/bin/bash
# One parameterised GPU session (run under gpurun from the repo root); replaces the per-round
# ab_cmd*/gpu_cmd* one-offs.  Everything is opt-in through the environment:
#   TESTS=none|quick|all     pytest -m "gpu and not slow" | -m gpu  (default none)
#   VARIANTS="v1 v2"         A/B builds paper_1511_06441_b200/libwcsp_<v>.so against the base build
#                            (build them first: python -m paper_1511_06441_b200.build -DNAME=val --out=...)
#   WS="C3 C2"               workloads timed by scripts/ab_bench.sh (bench.py's own timing, 2 reps)
#   VSLABS="2 4"             C3 cut into virtual slabs (peer halo), per variant
#   PHASE=C3                 per-phase breakdown (scripts/ab_phase.sh) of the variants on that workload
#   OUT=gpurun_out/ab        log prefix
OUT=${OUT:-gpurun_out/ab}
mkdir -p "$(dirname "$OUT")"
case "${TESTS:-none}" in
  quick) timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > "$OUT.tests.log" 2>&1; echo "tests=$?";;
  all)   timeout 1800 python -m pytest tests -m gpu -x -q > "$OUT.tests.log" 2>&1; echo "tests=$?";;
esac
for v in base ${VARIANTS}; do
  if [ "$v" != base ] && [ -n "${PARITY}" ]; then
    echo "## parity $v $(WCSP_LIB=paper_1511_06441_b200/libwcsp_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m 'gpu and not slow' -x -q 2>&1 | tail -1)"
  fi
done
[ -n "${WS}" ] && VARIANTS="${VARIANTS}" WS="${WS}" bash scripts/ab_bench.sh | tee "$OUT.bench.log"
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then lib=paper_1511_06441_b200/libwcsp.so; else lib=paper_1511_06441_b200/libwcsp_$v.so; fi
  for k in ${VSLABS}; do
    echo "== vslabs $k $v $(WCSP_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 3 --vslabs $k --halo peer --no-cpu-baseline --e2e-steps 0 2>/dev/null | grep '^{' | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["solve"]["F1"], d["solve"]["edge_updates"])')"
  done
done | tee -a "$OUT.bench.log"
[ -n "${PHASE}" ] && W=${PHASE} VARIANTS="${VARIANTS}" bash scripts/ab_phase.sh | tee "$OUT.phase.log"
echo done
