#!/bin/bash
# v14 A/B: events per lane in flight in the fire (WCSP_FIRE_ITEMS 6, 12) and no L2 cache-policy hints
VARIANTS="fi6 fi12 noh" WS="C3 C2" bash scripts/ab_bench.sh
