#!/bin/bash
# A/B of one runtime switch (an environment variable read by libwcsp) with bench.py's own timing.
#   VAR=WCSP_HYB_SPLIT VALS="0 1" WS="C3 C2 C3s C4" REPS=2 BIG="C5z8" bash scripts/ab_env.sh
# prints "== <workload> <VAR>=<val> rep<k> ms/solve frac edge_updates retries"; BIG workloads run once.
VAR=${VAR:?VAR} ; VALS=${VALS:-"0 1"} ; REPS=${REPS:-2}
one() {   # workload val rep steps
  env "$VAR=$2" timeout 900 python bench.py --workload "$1" --steps "$4" --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null |
    grep '^{' | python -c 'import sys,json; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"], d["solve"]["edge_updates"], d["solve"].get("retries", 0))' |
    sed "s/^/== $1 $VAR=$2 rep$3 /"
}
for w in ${WS:-C3 C2}; do
  for rep in $(seq 1 "$REPS"); do
    for val in $VALS; do one "$w" "$val" "$rep" 5; done
  done
done
for w in ${BIG}; do
  for val in $VALS; do one "$w" "$val" 1 2; done
done
