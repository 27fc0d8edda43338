#!/bin/bash
# A/B: per-phase breakdown of libwcsp.so variants (WCSP_LIB) on one workload.
# VARIANTS: names of paper_1511_06441_b200/libwcsp_<name>.so builds; ENVS: extra "VAR=value" runs of the base build.
W=${W:-C3}
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then lib=paper_1511_06441_b200/libwcsp.so; else lib=paper_1511_06441_b200/libwcsp_$v.so; fi
  echo "== $v"; WCSP_L2_PERSIST=0 WCSP_LIB=$lib python scripts/phase_breakdown.py $W wheel 2>&1 | grep '"cycle_ms"'
done
for e in ${ENVS}; do
  echo "== env $e"; env WCSP_L2_PERSIST=0 ${e//:/ } python scripts/phase_breakdown.py $W wheel 2>&1 | grep '"cycle_ms"'
done
