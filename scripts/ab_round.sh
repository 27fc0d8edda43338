echo "== base parity"; timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -1
for w in C3 C2 C3s C4; do W=$w VARIANTS="prev" bash scripts/ab_phase.sh 2>&1 | tail -4; done
