import sys, os
sys.path.insert(0, os.getcwd())
from bench import workload_instance
from paper_1511_06441_b200 import wcsp
for w in ("C3", "C2", "C3s", "P6-125", "C4"):
    inst, _ = workload_instance(w, 0)
    with wcsp.Solver(inst, engine="wheel") as s:
        r1 = s.solve(); r2 = s.solve()
    print(w, "first solve launches", r1.kernel_launches, "cap", r1.phantom_capacity, "second", r2.kernel_launches, flush=True)
