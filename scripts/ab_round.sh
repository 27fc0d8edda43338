for w in C3 C2; do W=$w VARIANTS="QPCAP4096 QPCAP3584" bash scripts/ab_phase.sh 2>&1 | tail -6; done
