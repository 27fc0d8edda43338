echo "== wf parity"; WCSP_LIB=paper_1511_06441_b200/libwcsp_wf.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "mid_sizes or fixtures or repeats or C1 or extreme or peer" 2>&1 | tail -1
for w in C3 C2 C3s P6-125 C4; do W=$w VARIANTS="wf" bash scripts/ab_phase.sh 2>&1 | tail -4; done
