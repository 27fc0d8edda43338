"""Write tests/golden/mbind.json: the binding budget of each
bench/test workload, M_bind = floor((F2_min + F2_lex)/2) + 1 (SURVEY §8
notation), from the CPU oracle's tier-3 Dijkstras ONLY (oracle/), never from
the CUDA path.  F2_min = min weight of an A->B path; F2_lex = weight of the
lexicographically fastest path.  Usage: python scripts/make_mbind.py C2 C3 --seeds 0-7
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1511_06441_b200 import instances as I  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "mbind.json")
SHAPES = {"C2": (1024, 1024), "C3": (256, 256, 256), "C3s": (128, 128, 128), "C5": (1024, 1024, 1024),
          # one z-slab of C5 at 8 GPUs (1024 x 1024 x 128): the DRAM-resident per-GPU regime
          "C5z8": (1024, 1024, 128),
          # §6 protocol: water on the cube's boundary, B = the centre vertex
          "P6-50": (50, 50, 50), "P6-75": (75, 75, 75), "P6-100": (100, 100, 100), "P6-125": (125, 125, 125)}


def main():
    args = sys.argv[1:]
    seeds = range(0, 5)
    if "--seeds" in args:
        a, b = args[args.index("--seeds") + 1].split("-")
        seeds = range(int(a), int(b) + 1)
    names = [a for a in args if a in SHAPES]
    table = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for name in names:
        for seed in seeds:
            key = f"{name}/{seed}"
            if key in table:
                continue
            t0 = time.time()
            if name.startswith("P6"):
                inst = I.grid_instance(SHAPES[name], seed, 1, 10, "boundary", "centre", I.M_INF, name)
            else:
                inst = I.config_face(SHAPES[name], seed, I.M_INF)
            lo, hi = oracle.solve_lex(inst, 1), oracle.solve_lex(inst, 0)
            table[key] = {"shape": list(SHAPES[name]), "seed": seed, "F2_min": lo.F2, "F1_at_F2min": lo.F1,
                          "F2_lex": hi.F2, "F1_lex": hi.F1, "M_bind": (lo.F2 + hi.F2) // 2 + 1,
                          "source": "oracle.solve_lex modes 1 and 0 (scripts/make_mbind.py)"}
            print(key, table[key], f"{time.time() - t0:.1f}s", flush=True)
            json.dump(table, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
