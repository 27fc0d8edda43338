"""Counters of single-device and peer-halo runs against oracle tier 5 on a few instances."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
from paper_1511_06441_b200 import instances as I, wcsp
def cnt(r): return (r.cycles, r.edge_updates, r.arrivals, r.triggered, r.phantoms_created, r.lanes_started, r.relabels)
for inst in [I.config_face((48, 48, 48), 0, 260), I.config_face((40, 40, 40), 3, 230)]:
    m, mc = oracle.solve_model(inst)
    want = (mc.cycles, mc.work, mc.arrivals, mc.triggered, mc.created, mc.started, mc.relabels)
    out = {"model": want}
    for eng in ("wheel", "persistent"):
        out[eng] = cnt(wcsp.solve(inst, engine=eng))
    out["peer3"] = cnt(wcsp.solve(inst, engine="wheel", slabs=3, halo="peer"))
    for k, v in out.items():
        print(inst.shape, k, v, "OK" if v == want else "DIFF", flush=True)
