# SPDX-License-Identifier: Apache-2.0
"""solve_exact on the GPU (csrc/exact.cu) against the reference's own
solve_exact (the memoised DFS of proj/src/solver.cpp:101-489, run through the
unmodified compiled library oracle/_ref): the same status, the same objective
bits AND the same optimal schedule — the tail_less winner (cost, sum R,
sum S, bit string; solver.cpp:87-92), so twin optima resolve identically.

Pins: tests/golden/exact_pins.json (scripts/gen_exact_pins.py: the
reference's test_solver.cpp fixtures, fig2 under both hazards, energy caps,
24 random DAGs x 3 budgets x 2 hazards) and tests/golden/exact_small.json
(scripts/gen_exact_golden.py: 157 random tight-budget cases)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_problem_text

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2212_09290_b200 as xe  # noqa: E402

STATUS = {"Optimal": "optimal", "Infeasible": "infeasible"}


def _cases(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)["cases"]


def _check(c, p, r):
    assert r.status == STATUS[c["status"]], (c.get("tag", c), r)
    if c["status"] == "Optimal":
        assert r.objective == c["objective"], (c.get("tag"), r.objective, c["objective"])
        got = r.cube
        want = np.asarray(c["cube"], np.uint32)
        assert np.array_equal(got, want), (c.get("tag", c), got.tolist(), want.tolist())
        # the tail_less keys are the cube's bit counts
        R, S = np.split(want, 2)
        assert r.sum_r == int(sum(bin(int(x)).count("1") for x in R))
        assert r.sum_s == int(sum(bin(int(x)).count("1") for x in S))


def test_reference_pins_same_schedule():
    bad = []
    for c in _cases("exact_pins.json"):
        p = xe.Problem.from_json(c["doc"])
        if c["budgets"]:
            p = p.with_budgets(c["budgets"])
        r = xe.solve_exact(p, xe.ModelOptions(strict_free=c["strict"], energy=c["energy"]))
        try:
            _check(c, p, r)
        except AssertionError as ex:
            bad.append(str(ex)[:300])
    assert not bad, bad[:4]


def test_random_small_same_schedule_as_reference():
    from bench import configs
    bad = []
    for c in _cases("exact_small.json"):
        p = xe.Problem.from_json(configs.random_small_doc(c["seed"], c["D"])).with_budgets([c["budget"]] * c["D"])
        r = xe.solve_exact(p)
        try:
            _check(c, p, r)
        except AssertionError as ex:
            bad.append(str(ex)[:300])
    assert not bad, bad[:4]


def test_optimum_peaks_within_budget_and_rescored():
    # the optimal schedule re-scored by the batched evaluator: the search's
    # cost is objective_value of the completion (fill_solution, solver.cpp:
    # 439-446), peaks within the budgets, check_assignment clean
    from paper_2212_09290_b200 import _lib
    for name in ("fig2", "chain_lowmem"):
        p = xe.Problem.from_json(golden_problem_text(name))
        r = xe.solve_exact(p)
        ev = xe.evaluate_cubes(p, torch.from_numpy(r.cube.view(np.int32)[None].copy()).cuda())
        assert ev.obj.item() == r.objective
        assert (ev.peak.cpu().numpy()[0] <= p.arrays()["budget_bytes"]).all()
        assert (int(ev.flags.item()) & (_lib.F_CHECK_MASK | _lib.F_BUDGET)) == 0


def test_limits():
    p = xe.Problem.from_json(golden_problem_text("fig2"))
    full = xe.solve_exact(p)
    assert full.status == "optimal" and full.nodes > 1000
    assert xe.solve_exact(p, node_limit=1).status == "limit"
    part = xe.solve_exact(p, node_limit=3000)
    assert part.status == "limit" and part.nodes <= 3001
    assert xe.solve_exact(p, time_limit_ms=0).status == "limit"


def test_too_large():
    doc = {"name": "c33", "devices": [{"id": "a", "budget_bytes": 1 << 30}, {"id": "b", "budget_bytes": 1 << 30}],
           "operators": [{"name": f"o{i}", "output_bytes": 1 << 20, "costs_ms": {"a": 1.0, "b": 1.0}}
                         for i in range(33)],
           "edges": [[i - 1, i] for i in range(1, 33)],
           "links": [{"from": "*", "to": "*", "latency_ms": 0.125, "bytes_per_ms": 1 << 30}]}
    with pytest.raises(xe.XeError) as ei:
        xe.solve_exact(xe.Problem.from_json(json.dumps(doc)))
    assert "TooLarge" in str(ei.value)


def test_upper_bound_prunes_without_changing_the_schedule():
    # a known schedule's cost as the bound: fewer states, same tail_less winner
    p = xe.Problem.from_json(golden_problem_text("fig2"))
    a = xe.solve_exact(p)
    b = xe.solve_exact(p, upper_bound=a.objective)
    assert b.status == "optimal" and b.objective == a.objective and np.array_equal(a.cube, b.cube)
    assert b.states <= a.states
