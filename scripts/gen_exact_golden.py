# SPDX-License-Identifier: Apache-2.0
"""The reference's exact optimum (solve_exact, the memoised DFS of
proj/src/solver.cpp:449-489, run through the UNMODIFIED compiled library
oracle/_ref) on seeded small random problems under tight memory budgets
-> tests/golden/exact_small.json, the pins of tests/test_search_gpu.py's
random sweep.  Run here (where /root/reference exists):
    python scripts/gen_exact_golden.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import xo  # noqa: E402
from bench import configs  # noqa: E402

STATUS = {0: "Optimal", 1: "Infeasible", 2: "LimitReached"}


def main():
    R = xo.Ref()
    out = {"solver": "reference solve_exact (oracle/_ref)", "cases": []}
    for seed in range(1, 31):
        for D in (2, 3):
            text = configs.random_small_doc(seed, D)
            rp = R.load(text)
            a = rp.arrays()
            full = int(a.mass.sum())
            for pct in (100, 60, 45):
                b = [xo.budget_percent(full, pct)] * D
                t0 = time.time()
                st, obj, cube, nodes = rp.solve_exact(D, a.T, budgets=b, node_limit=5_000_000)
                dt = time.time() - t0
                if STATUS[st] == "LimitReached":
                    continue
                out["cases"].append({"seed": seed, "D": D, "pct": pct, "budget": b[0], "T": a.T,
                                     "status": STATUS[st], "objective": obj if st == 0 else None,
                                     "nodes": nodes, "seconds": round(dt, 3),
                                     "cube": [int(x) for x in cube] if st == 0 else None})
                print(seed, D, pct, a.T, STATUS[st], obj, nodes, f"{dt:.2f}s", flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "exact_small.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
