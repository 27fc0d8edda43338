echo "== base parity"; timeout 900 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -1
echo "== QP_CAP256 parity"; WCSP_LIB=paper_1511_06441_b200/libwcsp_QP_CAP256.so timeout 600 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -1
for w in C3 C2 C3s P6-125; do W=$w VARIANTS="prev" bash scripts/ab_phase.sh 2>&1 | tail -4; done
