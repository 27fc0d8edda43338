"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck), one tool per run:
    compute-sanitizer --tool <tool> --error-exitcode 9 python scripts/sanitize_cases.py [quick]
Fixtures B and D (§2 mechanisms), C1b, a 24^3 face-to-face grid and a checkerboard
(staging overflow) on every engine, the 2-slab copy and peer halos, and a wide-label budget;
each checked against the oracle so a silent corruption also fails."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1511_06441_b200 import instances as I  # noqa: E402
from paper_1511_06441_b200 import wcsp  # noqa: E402

quick = "quick" in sys.argv
cases = [I.fixture_B(), I.fixture_D(), I.config_C1(3, 65), I.config_face((24, 24, 24), 2, 150)]
if not quick:
    chk = I.grid_instance((32, 32, 16), 4, 1, 10, "checker", "corner1", 200, "checker")
    cases.append(chk.with_sets(maskA=chk.maskA & (1 - chk.maskB)))
runs = [("persistent", {}), ("stepped", {}), ("wheel", {}), ("wheel_stepped", {}),
        ("wheel", {"slabs": 2, "halo": "copy"}), ("wheel", {"slabs": 2, "halo": "peer"})]
bad = 0
for inst in cases:
    want = oracle.solve_pruned(inst).key()
    for engine, kw in runs:
        if kw.get("slabs", 0) > inst.shape[-1]:
            continue
        r = wcsp.solve(inst, engine=engine, **kw)
        ok = r.key() == want
        bad += not ok
        print(f"{inst.name:>12} {engine:>13} {kw}: {r.key()} {'ok' if ok else 'MISMATCH ' + str(want)}", flush=True)
# wide labels (M > 65533): f2 near the u8 top
f1, _ = I.grid_values((120, 6), 1, 1, 10)
_, f2 = I.grid_values((120, 6), 2, 200, 255)
f2[f1 == 0] = 0
wide = I.Instance((120, 6), f1, f2, I.set_mask((120, 6), "face0"), I.set_mask((120, 6), "face1"), 70000, None, "wide")
for engine in ("persistent", "stepped"):
    r = wcsp.solve(wide, engine=engine)
    ok = r.key() == oracle.solve_pruned(wide).key()
    bad += not ok
    print(f"{'wide':>12} {engine:>13}: {r.key()} {'ok' if ok else 'MISMATCH'}", flush=True)
print("mismatches:", bad)
sys.exit(1 if bad else 0)
