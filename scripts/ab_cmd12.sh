#!/bin/bash
# v12 A/B: two-level grid-barrier arrivals (WCSP_BAR_GROUPS) and barrier poll sleep (WCSP_BAR_SLEEP)
WCSP_LIB=paper_1511_06441_b200/libwcsp_bg8sl0.so timeout 400 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q 2>&1 | tail -2
VARIANTS="bg8 bg16 sl0 bg8sl0" WS="C2 C4 C3" bash scripts/ab_bench.sh
