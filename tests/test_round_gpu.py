# SPDX-License-Identifier: Apache-2.0
"""K4 rounding/generator: candidates are valid for EQ8/EQ9/EQ11/EQ12 and the
fixed-zero triangles by construction (checked by the CPU oracle), and a
candidate is a pure function of (seed, global index)."""
import numpy as np
import pytest

from conftest import golden_problem_text
from oracle import xo
from bench import configs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200 import _lib  # noqa: E402

STRUCTURAL = _lib.F_FIXED_ZERO | _lib.F_EQ8 | _lib.F_EQ9 | _lib.F_EQ11 | _lib.F_EQ12 | _lib.F_EQ16_HI


@pytest.mark.parametrize("name", ["fig2", "vgg16", "resnet50", "unet"])
def test_rounded_candidates_valid_by_construction(oracle, name):
    text = golden_problem_text(name) if name == "fig2" else configs.CONFIGS[name]()
    a = xo.arrays_from_json(text)
    prob = xe.Problem.from_json(text)
    n = 64 if name in ("resnet50", "unet") else 500
    cubes = xe.round_cubes(prob, n, seed=11, edits=3, perturb=0.0).cpu().numpy().view(np.uint32)
    o, p, f = oracle.eval_cubes(a, cubes)
    assert ((f & STRUCTURAL) == 0).all(), [hex(x) for x in f[(f & STRUCTURAL) != 0][:5]]
    # recompute edits actually happen
    from cubegen import unpack
    R, S = unpack(cubes, a.D, a.T)
    assert R.sum(axis=(1, 2, 3)).max() > a.T


def test_round_is_index_deterministic():
    prob = xe.Problem.from_json(configs.vgg16_doc())
    whole = xe.round_cubes(prob, 1000, seed=5, first=0)
    parts = torch.cat([xe.round_cubes(prob, 300, seed=5, first=0),
                       xe.round_cubes(prob, 700, seed=5, first=300)])
    assert torch.equal(whole, parts)
    other = xe.round_cubes(prob, 1000, seed=6, first=0)
    assert not torch.equal(whole, other)


def test_perturbation_rate():
    text = configs.vgg16_doc()
    prob = xe.Problem.from_json(text)
    cubes = xe.round_cubes(prob, 20000, seed=3, perturb=0.1)
    r = xe.evaluate_cubes(prob, cubes)
    f = r.flags.cpu().numpy().view(np.uint32)
    bad = ((f & STRUCTURAL) != 0).mean()
    assert 0.02 < bad < 0.12  # single flips break a structural family most of the time


def test_local_search_neighbours(oracle):
    """xe_mutate_cubes: neighbours of an incumbent are index-deterministic,
    differ from it, keep the fixed-zero triangles, and the oracle agrees with
    the GPU evaluation of every neighbour."""
    text = configs.vgg16_doc()
    a = xo.arrays_from_json(text)
    prob = xe.Problem.from_json(text)
    base = xe.round_cubes(prob, 1, seed=4)[0]
    nb = xe.mutate_cubes(prob, base, 512, seed=9, edits=2)
    again = torch.cat([xe.mutate_cubes(prob, base, 200, seed=9, edits=2),
                       xe.mutate_cubes(prob, base, 312, seed=9, first=200, edits=2)])
    assert torch.equal(nb, again)
    changed = (nb != base.unsqueeze(0)).any(dim=1).float().mean().item()
    assert changed > 0.5
    cubes = nb.cpu().numpy().view(np.uint32)
    o, p, f = oracle.eval_cubes(a, cubes)
    assert ((f & _lib.F_FIXED_ZERO) == 0).all()
    r = xe.evaluate_cubes(prob, nb)
    assert np.array_equal(r.obj.cpu().numpy().view(np.int64), o.view(np.int64))
    assert np.array_equal(r.peak.cpu().numpy(), p)
