L=paper_1511_06441_b200
q() { WCSP_L2_PERSIST=0 timeout 300 python scripts/phase_breakdown.py $1 wheel 2>&1 | grep '"cycle_ms"' | python -c 'import sys,json; l=sys.stdin.read(); d=json.loads(l[l.index("{"):]); print("cycle_ms %.2f arrive %.2f treat %.2f other %.2f spread a/t %.2f/%.2f" % (d["cycle_ms"], d["arrive_ms"], d["treat_ms"], d["other_ms"], d["arrive_spread_ms"], d["treat_spread_ms"]))'; }
for w in C3 C2; do for rep in 1 2; do
 echo "== $w base $(q $w)"
 echo "== $w win32/32 $(WCSP_LIB=$L/libwcsp_win32.so WCSP_WIN_WORDS=32 q $w)"
 echo "== $w win32/16 $(WCSP_LIB=$L/libwcsp_win32.so WCSP_WIN_WORDS=16 q $w)"
 echo "== $w qp4k $(WCSP_LIB=$L/libwcsp_qp4k.so q $w)"
done; done
