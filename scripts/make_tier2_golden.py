"""Write tests/golden/tier2_full.json: oracle tier 2 (oracle/wcsp_oracle.c
orc_pruned — time-ordered label setting on remaining quality, a definition-based
solver independent of the paper's cycle) run IN FULL on the bench
configuration(s), with the CPU time it took on this host.  Calls only oracle/
(and the seeded instance generator).

    python scripts/make_tier2_golden.py C3        # configs[2], seed 0, M_bind
"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1511_06441_b200 import instances as I  # noqa: E402

SHAPES = {"C2": (1024, 1024), "C3": (256, 256, 256), "C3s": (128, 128, 128)}
OUT = os.path.join(ROOT, "tests", "golden", "tier2_full.json")
MBIND = json.load(open(os.path.join(ROOT, "tests", "golden", "mbind.json")))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main(names):
    table = json.load(open(OUT)) if os.path.exists(OUT) else {}
    table["_source"] = ("scripts/make_tier2_golden.py: oracle.solve_pruned (tier 2) in full on "
                        "instances.config_face(shape, seed) at M = M_bind (tests/golden/mbind.json)")
    for name in names:
        key = f"{name}/0"
        M = MBIND[key]["M_bind"]
        inst = I.config_face(SHAPES[name], 0, M, name=name)
        t0 = time.perf_counter()
        r = oracle.solve_pruned(inst)
        dt = time.perf_counter() - t0
        table[key] = {"M": M, "key": list(r.key()), "flows": r.work, "event_times": r.cycles,
                      "cpu_seconds": round(dt, 1), "cores": 1, "cpu": cpu_model()}
        print(key, table[key], flush=True)
        json.dump(table, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C3"])
