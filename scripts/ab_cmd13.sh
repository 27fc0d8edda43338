#!/bin/bash
# v13 A/B: merged treat rounds (WCSP_ROUND_MERGE = 2, 4)
for v in rm2 rm4; do echo "## parity $v"; WCSP_LIB=paper_1511_06441_b200/libwcsp_$v.so timeout 400 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q 2>&1 | tail -2; done
VARIANTS="rm2 rm4" WS="C3 C2 C3s" bash scripts/ab_bench.sh
