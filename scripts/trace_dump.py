"""Dump the per-cycle trace of one solve (default engine) to gpurun_out/trace_<W>.npz."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from bench import workload_instance
from paper_1511_06441_b200 import wcsp
w = sys.argv[1] if len(sys.argv) > 1 else "C3"
inst, _ = workload_instance(w, 0)
with wcsp.Solver(inst, engine="wheel", trace_cap=100000) as s:
    s.solve()
    r = s.solve()
    tr = s.trace()
os.makedirs("gpurun_out", exist_ok=True)
np.savez(f"gpurun_out/trace_{w}.npz", **{k: np.asarray(v) for k, v in tr.items()})
print(w, r.cycle_ms, len(tr["t"]))
