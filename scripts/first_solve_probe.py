"""Which structure (if any) overflows on a fresh handle's first solve (retries, capacity) — C3."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import workload_instance
from paper_1511_06441_b200 import wcsp
inst, _ = workload_instance(sys.argv[1] if len(sys.argv) > 1 else "C3", 0)
with wcsp.Solver(inst, engine="wheel") as s:
    for i in range(3):
        r = s.solve()
        print(json.dumps({"solve": i, "retries": r.retries, "capacity": r.phantom_capacity, "cycle_ms": r.cycle_ms,
                          "device_ms": r.device_ms, "launches": r.kernel_launches}), flush=True)
