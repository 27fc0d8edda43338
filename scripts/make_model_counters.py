"""Write tests/golden/model_counters.json: oracle tier 5 (the paper's cycle run
sequentially, oracle.solve_model) at BASELINE.json's full sizes, so the GPU
tests can compare the metric's numerator (edge_updates) and every other work
counter bit-exactly without re-running a 4-45 minute sequential simulation.

Calls only oracle/ and the instance generator.  Usage:
    python scripts/make_model_counters.py C2/0 C3/0
"""
import dataclasses
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1511_06441_b200 import instances as I  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "model_counters.json")
MBIND = json.load(open(os.path.join(ROOT, "tests", "golden", "mbind.json")))
SHAPES = {"C2": (1024, 1024), "C3": (256, 256, 256), "C3s": (128, 128, 128)}


def main(keys):
    out = json.load(open(OUT)) if os.path.exists(OUT) else {
        "_source": "scripts/make_model_counters.py: oracle.solve_model (tier 5, jump time) on "
                   "instances.config_face(shape, seed) at M = M_bind (tests/golden/mbind.json)"}
    for key in keys:
        name, seed = key.split("/")
        inst = I.config_face(SHAPES[name], int(seed), I.M_INF).with_M(MBIND[key]["M_bind"])
        t0 = time.time()
        r, c = oracle.solve_model(inst)
        out[key] = {"M": inst.M, "key": list(r.key()), "counters": dataclasses.asdict(c),
                    "cpu_seconds": round(time.time() - t0, 1)}
        print(key, out[key], flush=True)
        json.dump(out, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C2/0"])
