echo "== w32 parity"; WCSP_WIN_WORDS=32 WCSP_LIB=paper_1511_06441_b200/libwcsp_w32.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "mid_sizes or fixtures or repeats or C1" 2>&1 | tail -1
for w in C3 C2; do W=$w ENVS="WCSP_LIB=paper_1511_06441_b200/libwcsp_w32.so:WCSP_WIN_WORDS=32" bash scripts/ab_phase.sh 2>&1 | tail -4; done
