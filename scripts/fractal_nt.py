"""Theorem 2 measurement (SURVEY f3 / reading R27): N_t = active
vertices with |x| <= t at time t on the fractal environment omega_k (t = 2^k),
M = infinity, unit time, B moved to (0, t + 1) so the run passes time t.  Compared
with the continuum bound (4/15) k t — reported, not asserted
(the staircase rasterisation does not grow the frontier)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_06441_b200 import instances as I  # noqa: E402
from paper_1511_06441_b200 import wcsp  # noqa: E402

rows = []
for k in range(3, int(sys.argv[1]) + 1 if len(sys.argv) > 1 else 13):
    t = 1 << k
    f = I.fractal_instance(k, B=[(0, t + 1)])
    with wcsp.Solver(f, engine="persistent", time_mode="unit", trace_cap=t + 8) as s:
        r = s.solve()
        tr = s.trace()
    idx = [i for i, tt in enumerate(tr["t"]) if tt == t + 1]
    nt = int(tr["active_vertices"][idx[0]]) if idx else None      # active after time t (top of cycle t+1)
    row = {"k": k, "t": t, "N_t": nt, "bound_4_15_k_t": round(4 / 15 * k * t, 1), "F1_to_(0,t+1)": r.F1,
           "solve_ms": round(r.device_ms, 3), "cycles": r.cycles}
    rows.append(row)
    print(json.dumps(row), flush=True)
