timeout 700 python -m pytest tests -m "gpu and not slow" -x -q 2>&1 | tail -2
WCSP_LIB=paper_1511_06441_b200/libwcsp_bitloop.so timeout 700 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q 2>&1 | tail -2
VARIANTS="prev bitloop" WS="C3 C2 C3s" bash scripts/ab_quick.sh
