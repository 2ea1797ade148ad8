# SPDX-License-Identifier: Apache-2.0
"""Exact optima WITH their schedules from the reference's solve_exact (the
memoised DFS of proj/src/solver.cpp:101-489, run through the UNMODIFIED
compiled library oracle/_ref) -> tests/golden/exact_pins.json, the pins of
tests/test_exact_gpu.py: status, objective, the optimal (R, S) cube (the
tail_less winner, solver.cpp:87-92) and the node count.

Cases: the reference's own test_solver.cpp fixtures (chain3 and its 8 / 3
MiB budgets :66-97, fig2 :99-119, the chain_lowmem sweep and boundaries
:121-153, the energy cap :223-237 and alpha :239-249), both hazard modes on
fig2, and seeded random DAGs (configs.random_small_doc) under the default
and the strict hazard at 100 / 60 / 45 % of save-all.  Run here (where
/root/reference exists):  python scripts/gen_exact_pins.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import xo  # noqa: E402
from bench import configs  # noqa: E402

MiB = 1 << 20
STATUS = {0: "Optimal", 1: "Infeasible", 2: "LimitReached"}


def golden_text(name):
    with open(os.path.join(ROOT, "tests", "golden", "problems", name + ".json")) as f:
        return f.read()


def main():
    R = xo.Ref()
    cases = []

    def run(tag, text, budgets=None, strict=False, energy=False):
        rp = R.load(text)
        a = rp.arrays()
        st, obj, cube, nodes = rp.solve_exact(a.D, a.T, strict=strict, energy=energy, budgets=budgets,
                                              node_limit=20_000_000)
        if STATUS[st] == "LimitReached":
            print("skip (limit)", tag)
            return
        cases.append({"tag": tag, "doc": text, "budgets": budgets, "strict": strict, "energy": energy,
                      "status": STATUS[st], "objective": obj if st == 0 else None, "nodes": nodes,
                      "cube": [int(x) for x in cube] if st == 0 else None})
        print(tag, STATUS[st], obj, nodes, flush=True)

    c3 = golden_text("chain3")
    run("chain3", c3)
    run("chain3@8MiB", c3, [8 * MiB])
    run("chain3@3MiB", c3, [3 * MiB])
    f2 = golden_text("fig2")
    run("fig2", f2)
    run("fig2/strict", f2, strict=True)
    lm = golden_text("chain_lowmem")
    full = 34 * MiB
    for pct in (100, 65, 50, 35, 25):
        run(f"chain_lowmem@{pct}", lm, [xo.budget_percent(full, pct)])
    for b in (10 * MiB, 9 * MiB, 8 * MiB, 4 * MiB - 1):
        run(f"chain_lowmem@{b}", lm, [b])
    fe = golden_text("fig2_energy")
    run("fig2_energy", fe, energy=True)
    doc = json.loads(fe)
    doc["energy"].pop("device_limit")
    run("fig2_energy/nocap", json.dumps(doc), energy=True)
    doc = json.loads(c3)
    dev = doc["devices"][0]["id"]
    doc["energy"] = {"alpha": 1.0, "q_joules": {dev: [2.0, 3.0, 4.0]}, "board_joules": 0.0}
    run("chain3/alpha1", json.dumps(doc), energy=True)
    for seed in range(1, 13):
        for D in (2, 3):
            text = configs.random_small_doc(seed, D)
            a = R.load(text).arrays()
            full = int(a.mass.sum())
            for pct in (100, 60, 45):
                for strict in (False, True):
                    run(f"rand{seed}/D{D}/{pct}/{'strict' if strict else 'default'}", text,
                        [xo.budget_percent(full, pct)] * D, strict=strict)
    with open(os.path.join(ROOT, "tests", "golden", "exact_pins.json"), "w") as f:
        json.dump({"solver": "reference solve_exact (oracle/_ref)", "cases": cases}, f, indent=0)


if __name__ == "__main__":
    main()
