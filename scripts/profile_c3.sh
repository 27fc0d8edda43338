#!/bin/bash
# Final-HEAD evidence for the default bench workload (run under gpurun from the repo root):
#   RUN=r02ag KERNEL=k_wheel_lag MANGLED=_ZN5wcspk11k_wheel_lagILi3ELi4EEEvNS_3DevE bash scripts/profile_c3.sh
# bench line (20 timed steps), ncu launch list, one `ncu --set full` capture of the timed cycle-kernel
# launch (report kept in /tmp: too large for gpurun_out) exported as per-line stall / instruction
# tables, raw and details pages.
RUN=${RUN:?RUN}; KERNEL=${KERNEL:-k_wheel_lag}; MANGLED=${MANGLED:?MANGLED}
O=gpurun_out/$RUN; mkdir -p "$O"
timeout 900 python bench.py --steps 20 --warmup 5 > "$O/bench_default.log" 2>&1; echo bench=$?
B="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
$B > "$O/plain.log" 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$O/launches_c3.csv" $B > "$O/ncu_launches.log" 2>&1; echo launches=$?
B1="python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline"
$B1 > "$O/plain1.log" 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on \
  -k "regex:$KERNEL" -s 1 -c 1 -o /tmp/prof_c3 $B1 > "$O/ncu.log" 2>&1; echo ncu=$?
python scripts/ncu_lines.py /tmp/prof_c3.ncu-rep "$KERNEL" "$MANGLED" 50 > "$O/lines_c3.txt" 2>&1
NCU_COL="Instructions Executed" python scripts/ncu_lines.py /tmp/prof_c3.ncu-rep "$KERNEL" "$MANGLED" 50 > "$O/instr_c3.txt" 2>&1
ncu -i /tmp/prof_c3.ncu-rep --page raw --csv > "$O/raw_c3.csv" 2>&1
ncu -i /tmp/prof_c3.ncu-rep --page details --csv > "$O/details_c3.csv" 2>&1
