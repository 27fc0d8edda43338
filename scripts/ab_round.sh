echo "== base parity"; timeout 600 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -1
for w in C3 C2 C3s P6-125 C4; do W=$w bash scripts/ab_phase.sh 2>&1 | tail -2; done
