for w in C2 C4 P6-125 C3; do W=$w ENVS="WCSP_LIST_MAX=0 WCSP_LIST_MAX=7000 WCSP_LIST_MAX=113000" bash scripts/ab_phase.sh 2>&1 | tail -8; done
