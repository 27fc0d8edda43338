#!/bin/bash
# A/B of libwcsp variants (VARIANTS) with bench.py's own timing (no trace), WS workloads, 2 alternating reps.
for w in ${WS:-C3 C2}; do
  for rep in 1 2; do
    for v in base ${VARIANTS}; do
      if [ "$v" = base ]; then lib=paper_1511_06441_b200/libwcsp.so; else lib=paper_1511_06441_b200/libwcsp_$v.so; fi
      echo "== $w $v rep$rep $(WCSP_LIB=$lib timeout 300 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | grep '^{' | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print("ms %.2f value %.4g" % (d["ms_per_step"], d["value"]))')"
    done
  done
done
