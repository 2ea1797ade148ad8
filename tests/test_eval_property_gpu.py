# SPDX-License-Identifier: Apache-2.0
"""Property sweep of the K2a evaluators against the CPU oracle (pinned to the
reference, tests/test_oracle_cpu.py) on random problems outside the fixture
shapes: T up to 64 (interleaved one-word kernel) and up to 140 (warp kernel),
D in 1..8 (every MAXD instantiation), non-dyadic costs (per-candidate objectives
within 1e-12 relative, the best-of-batch bit-exact), per-edge copy overrides, dst-unsorted edge orders (the ordered copy
walk), tight budgets (BUDGET / U_BOUND flags), strict and default hazards,
and an energy section.  Bit-exact objectives, peaks and flags."""
import json

import numpy as np
import pytest

from oracle import xo
import cubegen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200 import _lib  # noqa: E402

MiB = 1 << 20


def random_doc(seed, T, D, energy=False, sort_by_dst=False):
    rng = np.random.default_rng(seed)
    devs = [f"d{d}" for d in range(D)]
    ops, edges = [], []
    for i in range(T):
        costs = {dv: round(float(rng.uniform(0.01, 3.0)), 4) for dv in devs}
        if i == 0 and D > 1:
            costs = {devs[0]: 0.0}  # the pinned input: every other device prohibitive
        ops.append({"name": f"op{i}", "output_bytes": int(rng.integers(1, 9)) * MiB // 2, "costs_ms": costs})
        if i > 0:
            edges.append((int(rng.integers(max(0, i - 3), i)), i))
    for v in range(2, T):
        for _ in range(int(rng.integers(0, 3))):
            u = int(rng.integers(0, v))
            if (u, v) not in edges:
                edges.append((u, v))
    edges = sorted(edges, key=(lambda e: (e[1], e[0])) if sort_by_dst else (lambda e: e))
    full = sum(o["output_bytes"] for o in ops)
    ej = []
    for (u, v) in edges:
        if D > 1 and rng.random() < 0.2:
            ej.append({"src": u, "dst": v, "copy_ms": {f"{devs[0]}->{devs[1]}": round(float(rng.uniform(0.1, 2)), 3)}})
        else:
            ej.append([u, v])
    doc = {"name": f"prop{seed}", "devices": [{"id": dv, "budget_bytes": int(full * rng.uniform(0.3, 1.0))} for dv in devs],
           "operators": ops, "edges": ej,
           "links": [{"from": "*", "to": "*", "latency_ms": 0.05, "bytes_per_ms": 7.5e6}]}
    if energy:
        doc["energy"] = {"alpha": 0.5, "q_joules": {dv: [round(float(rng.uniform(0, 2)), 3) for _ in range(T)] for dv in devs},
                         "device_limit": {devs[-1]: 1.5}, "total_limit": 3.0, "board_joules": 0.25}
    return json.dumps(doc)


CASES = [(1, 40, 1), (2, 43, 2), (3, 64, 3), (4, 50, 4), (5, 33, 5), (6, 61, 8), (7, 17, 2), (8, 100, 3),
         (9, 140, 4), (10, 70, 2)]


@pytest.mark.parametrize("seed,T,D", CASES)
def test_random_problems_vs_oracle(oracle, seed, T, D):
    for sort_by_dst in (False, True):
        for energy in (False, True):
            text = random_doc(seed, T, D, energy=energy, sort_by_dst=sort_by_dst)
            a = xo.arrays_from_json(text)
            prob = xe.Problem.from_json(text)
            cubes = cubegen.mixed_cubes(a, 64 if T > 64 else 200, seed=seed, edits=3, random_frac=0.03)
            t = torch.from_numpy(cubes.view(np.int32)).cuda()
            for strict in (0, 1):
                opts = xe.ModelOptions(strict_free=bool(strict), energy=energy)
                r = xe.evaluate_cubes(prob, t, opts)
                torch.cuda.synchronize()
                o, p, f = r.obj.cpu().numpy(), r.peak.cpu().numpy(), r.flags.cpu().numpy().view(np.uint32)
                ro, rp, rf = oracle.eval_cubes(a, cubes, strict, energy)
                if energy or prob.objective_order_exact:
                    assert np.array_equal(o.view(np.int64), ro.view(np.int64)), (seed, strict, energy, sort_by_dst)
                else:  # per-timestep reassociation (test_eval_gpu.REL)
                    assert np.all(np.abs(o - ro) <= 1e-12 * np.abs(ro)), (seed, strict, sort_by_dst)
                valid = (rf & _lib.F_CHECK_MASK) == 0
                if valid.any():
                    idx = np.nonzero(valid)[0]
                    best = idx[np.argmin(ro[idx].view(np.int64))]
                    assert r.best_index == best and np.float64(r.best_obj).view(np.int64) == ro[best].view(np.int64)
                assert np.array_equal(p, rp)
                mask = 0xFFFF | _lib.F_DECODE
                assert np.array_equal(f & mask, rf & mask)
                comparable = ((rf & _lib.F_DECODE) != 0) & ((f & _lib.F_EQ12) == 0)
                assert np.array_equal((f & _lib.F_DECODE_FREED)[comparable], (rf & _lib.F_DECODE_FREED)[comparable])
