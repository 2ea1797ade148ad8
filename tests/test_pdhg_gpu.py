# SPDX-License-Identifier: Apache-2.0
"""K3 PDHG LP relaxation against HiGHS on the reference model
(tests/golden/lp_values.json, scripts/gen_lp_golden.py): objective within
1e-5 relative (the north-star tolerance), primal feasibility, bound overrides."""
import json
import os

import pytest

from conftest import GOLDEN, golden_problem_text
from bench import configs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2212_09290_b200 as xe  # noqa: E402

LP = json.load(open(os.path.join(GOLDEN, "lp_values.json")))


def problem(name):
    if name == "chain3":
        return xe.Problem.from_json(golden_problem_text("chain3"))
    if name.startswith("fig2_energy"):
        return xe.Problem.from_json(golden_problem_text("fig2_energy"))
    if name.startswith("fig2"):
        return xe.Problem.from_json(configs.fig2_doc())
    if name == "vgg16":
        return xe.Problem.from_json(configs.vgg16_doc())
    if name.startswith("chain_lowmem"):
        p = xe.Problem.from_json(golden_problem_text("chain_lowmem"))
        full = int(p.arrays()["output_bytes"].sum())
        return p.with_budgets([full * 25 // 100])
    if name.startswith("rand"):
        return xe.Problem.from_json(configs.random_small_doc(int(name[4:])))
    if name == "resnet50":
        return xe.Problem.from_json(configs.resnet50_doc())
    if name == "unet":
        return xe.Problem.from_json(configs.unet_doc())
    raise KeyError(name)


CASES = ["chain3", "chain_lowmem@25", "rand1", "rand2", "rand3", "rand4", "rand5",
         "fig2", "fig2_strict", "fig2_energy", "vgg16"]


@pytest.mark.parametrize("name", CASES)
def test_lp_objective_matches_highs(name):
    want = LP[name]["lp"]
    opts = xe.ModelOptions(strict_free=name.endswith("strict"), energy=name.endswith("energy"))
    m = xe.build_model(problem(name), opts)
    r = xe.pdhg_solve(m, tol=1e-7, max_iters=400000)
    assert r.converged, r
    assert r.certified, r  # the prohibitive-cost presolve is priced out by the final duals
    assert abs(r.primal_obj - want) <= 1e-5 * max(1.0, abs(want)), (r.primal_obj, want)
    assert abs(r.dual_obj - want) <= 1e-5 * max(1.0, abs(want)), (r.dual_obj, want)
    assert r.rel_primal_res <= 1e-6


def test_bound_overrides_fix_a_node():
    # fixing the diagonal of op 1 on the gpu can only raise the LP bound
    p = problem("fig2")
    m = xe.build_model(p)
    base = xe.pdhg_solve(m, tol=1e-7, max_iters=200000)
    h = m.to_host()
    lb = h["lb"].copy()
    T = 7
    col = (1 * T + 1) * T + 1  # R(d=1, t=1, i=1)
    lb[col] = 1.0
    node = xe.pdhg_solve(m, tol=1e-7, max_iters=200000, lb=lb, return_x=True)
    assert node.converged
    assert node.x[col] >= 1.0 - 1e-6
    assert node.primal_obj >= base.primal_obj - 1e-6


@pytest.mark.parametrize("name", ["resnet50", "unet"])
def test_large_lp(name):
    # configs 3 and 4 (HiGHS IPM goldens: scripts/gen_lp_golden.py --big / --unet)
    if name not in LP:
        pytest.skip(f"no HiGHS golden for {name} (scripts/gen_lp_golden.py)")
    want = LP[name]["lp"]
    m = xe.build_model(problem(name))
    r = xe.pdhg_solve(m, tol=1e-7, max_iters=1000000)
    assert r.certified
    assert abs(r.primal_obj - want) <= 1e-5 * abs(want), (r.primal_obj, want, r.iters)
