timeout 900 python -m pytest tests -m "gpu" -x -q 2>&1 | tail -2
for bps in 4 3; do echo "## blocks/SM $bps"; WCSP_BLOCKS_PER_SM=$bps VARIANTS="nobc" WS="C3 C2 C3s C4" bash scripts/ab_bench.sh; done
