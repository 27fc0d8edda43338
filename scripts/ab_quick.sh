#!/bin/bash
# A/B of libwcsp variants (VARIANTS) on workloads (WS), each run twice (alternating) to see noise.
for w in ${WS:-C3 C2}; do
  for rep in 1 2; do
    for v in base ${VARIANTS}; do
      if [ "$v" = base ]; then lib=paper_1511_06441_b200/libwcsp.so; else lib=paper_1511_06441_b200/libwcsp_$v.so; fi
      echo "== $w $v rep$rep $(WCSP_L2_PERSIST=0 WCSP_LIB=$lib timeout 300 python scripts/phase_breakdown.py $w wheel 2>&1 | grep '"cycle_ms"' | python -c 'import sys,json; l=sys.stdin.read(); d=json.loads(l[l.index("{"):]); print("cycle_ms %.2f arrive %.2f treat %.2f other %.2f spread a/t %.2f/%.2f tested %d created %d" % (d["cycle_ms"], d["arrive_ms"], d["treat_ms"], d["other_ms"], d["arrive_spread_ms"], d["treat_spread_ms"], d["tested"], d["created"]))')"
    done
  done
done
