#!/bin/bash
# v15 A/B: fire events per lane in the 4-blocks-per-SM build (16, 10 against 12)
VARIANTS="f16 f10" WS="C3 C3s" bash scripts/ab_bench.sh
