VARIANTS="fi4 qp2k fpf" WS="C3 C3s" bash scripts/ab_bench.sh
echo "## window words 8"; WCSP_WIN_WORDS=8 VARIANTS="" WS="C3" bash scripts/ab_bench.sh
