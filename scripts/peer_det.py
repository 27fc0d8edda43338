"""Determinism probe of the peer-halo slab engine: repeated solves of one instance."""
import sys, os, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_06441_b200 import instances as I, wcsp
insts = [I.config_face((48, 48, 48), 0, 260), I.config_face((32, 32, 32), 2, 200), I.config_face((64, 64), 1, 300)]
for inst in insts:
    r1 = wcsp.solve(inst, engine="wheel")
    base = (r1.cycles, r1.edge_updates, r1.arrivals, r1.triggered, r1.phantoms_created, r1.lanes_started, r1.relabels)
    for slabs in (2, 3, 5):
        cnt = collections.Counter()
        for _ in range(10):
            r = wcsp.solve(inst, engine="wheel", slabs=slabs, halo="peer")
            cnt[(r.key() == r1.key(), (r.cycles, r.edge_updates, r.arrivals, r.triggered, r.phantoms_created, r.lanes_started, r.relabels) == base)] += 1
        print(inst.shape, slabs, dict(cnt), flush=True)
