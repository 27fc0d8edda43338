timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
VARIANTS="nosteal" WS="C3 C2 C3s" bash scripts/ab_quick.sh
