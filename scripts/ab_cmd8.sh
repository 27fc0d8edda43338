timeout 700 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
VARIANTS="nobar prev m4div" WS="C3 C2 C3s C4" bash scripts/ab_bench.sh
