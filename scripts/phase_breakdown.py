"""Per-phase device-time breakdown of one solve (trace ns_arrive / ns_treat as seen by block 0)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import workload_instance  # noqa: E402
from paper_1511_06441_b200 import wcsp  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
engines = sys.argv[2:] or ["wheel", "persistent"]
inst, meta = workload_instance(wl, 0)
out = {}
for e in engines:
    with wcsp.Solver(inst, engine=e, trace_cap=100000) as s:
        s.solve()
        r = s.solve()
        tr = s.trace()
    na, nt = tr["ns_arrive"].sum() / 1e6, tr["ns_treat"].sum() / 1e6
    out[e] = {"cycle_ms": r.cycle_ms, "cycles": r.cycles, "arrive_ms": na, "treat_ms": nt,
              "other_ms": r.cycle_ms - na - nt, "tested": int(tr["tested"].sum()), "triggered": r.triggered,
              "arrivals": r.arrivals, "created": r.phantoms_created, "started": r.lanes_started,
              "max_cycle_us": float((tr["ns_arrive"] + tr["ns_treat"]).max() / 1e3),
              "arrive_spread_ms": float(tr["ns_arrive_spread"][1:].sum() / 1e6),
              "treat_spread_ms": float(tr["ns_treat_spread"][1:].sum() / 1e6)}
    print(wl, e, json.dumps(out[e]), flush=True)
    if e.startswith("wheel"):
        nd = tr["active_vertices"].astype(float)
        ev = tr["arrivals"].astype(float)
        m = nd > 0
        print("  runs per bucket: mean %.0f max %.0f; events per run: mean %.0f; cycles with < 4736 runs: %d of %d"
              % (nd[m].mean(), nd.max(), (ev[m] / nd[m]).mean(), int((nd < 4736).sum()), len(nd)))
        mid = len(nd) // 2
        print("  mid-run cycle:", {k: int(tr[k][mid]) for k in ("t", "active_vertices", "arrivals", "tested", "ns_arrive", "ns_treat")})
