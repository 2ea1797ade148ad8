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
    prob = xe.Problem.from_json(text).set_exact_objective()  # objective bits compared with the oracle
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


def canonical_saves_numpy(a, R):
    """Restatement of the canonical saves (xe_move_cubes): tensor u kept on
    the (lowest) device of its latest computation at every step t where its
    next need (a consumer computed, any device) comes before its next
    computation."""
    D, T = a.D, a.T
    cons = [[] for _ in range(T)]
    for s_, d_ in zip(a.src, a.dst):
        cons[s_].append(d_)
    comp = R.any(axis=0)  # [t][i]
    S = np.zeros_like(R)
    for u in range(T):
        need = comp[:, cons[u]].any(axis=1) if cons[u] else np.zeros(T, bool)
        nn = nc = T
        hold = np.zeros(T, bool)
        for t in range(T - 1, -1, -1):
            if comp[t, u]:
                nc = t
            if need[t]:
                nn = t
            hold[t] = nn < nc
        hd = -1
        for t in range(T):
            if comp[t, u]:
                hd = int(np.flatnonzero(R[:, t, u])[0])
            elif hd >= 0 and hold[t]:
                S[hd, t, u] = True
    return S


@pytest.mark.parametrize("name", ["fig2", "vgg16", "resnet50"])
def test_move_cubes_canonical_saves(oracle, name):
    from cubegen import unpack
    text = golden_problem_text(name) if name == "fig2" else configs.CONFIGS[name]()
    a = xo.arrays_from_json(text)
    prob = xe.Problem.from_json(text).set_exact_objective()  # objective bits compared with the oracle
    n = 32 if name == "resnet50" else 200
    base = xe.round_cubes(prob, n, seed=3, edits=4, perturb=0.0)
    canon = xe.move_cubes(prob, base, n, 0, max_moves=0)
    c = canon.cpu().numpy().view(np.uint32)
    R0, _ = unpack(base.cpu().numpy().view(np.uint32), a.D, a.T)
    R, S = unpack(c, a.D, a.T)
    assert np.array_equal(R, R0)  # no move: computations unchanged
    for k in range(n):
        assert np.array_equal(S[k], canonical_saves_numpy(a, R[k])), k
    # idempotent, and the K2 evaluation of canonical cubes matches the oracle bit for bit
    assert torch.equal(xe.move_cubes(prob, canon, n, 0, max_moves=0), canon)
    o, p, f = oracle.eval_cubes(a, c)
    r = xe.evaluate_cubes(prob, canon, valid_mask=0)
    assert np.array_equal(r.obj.cpu().numpy().view(np.int64), o.view(np.int64))
    assert np.array_equal(r.peak.cpu().numpy(), p)
    assert np.array_equal(r.flags.cpu().numpy().astype(np.uint32), f)
    # the rounding's structural validity survives (holders exist where needed)
    assert ((f & STRUCTURAL) == 0).all()


def test_move_cubes_neighbours(oracle):
    from cubegen import unpack
    a = xo.arrays_from_json(configs.vgg16_doc())
    prob = xe.Problem.from_json(configs.vgg16_doc()).set_exact_objective()  # objective bits compared with the oracle
    bases = xe.move_cubes(prob, xe.round_cubes(prob, 4, seed=9, edits=3, perturb=0.0), 4, 0, max_moves=0)
    nb = xe.move_cubes(prob, bases, 4 * 256, 21, first=0, max_moves=3)
    # pure function of (seed, index, base); chains map to blocks of 256
    assert torch.equal(nb, xe.move_cubes(prob, bases, 4 * 256, 21, first=0, max_moves=3))
    R, S = unpack(nb.cpu().numpy().view(np.uint32), a.D, a.T)
    Rb, _ = unpack(bases.cpu().numpy().view(np.uint32), a.D, a.T)
    changed = 0
    for k in range(nb.shape[0]):
        diff = int((R[k] != Rb[k // 256]).sum())
        changed += diff > 0
        assert np.array_equal(S[k], canonical_saves_numpy(a, R[k]))
    assert changed > 0.8 * nb.shape[0]
    # neighbours keep one diagonal computation per step and no R above the diagonal
    assert (R[:, :, np.arange(a.T), np.arange(a.T)].sum(axis=1) == 1).all()
    assert not np.triu(np.ones((a.T, a.T), bool), 1)[None, None].__and__(R).any()
    o, p, f = oracle.eval_cubes(a, nb.cpu().numpy().view(np.uint32), strict=True)
    r = xe.evaluate_cubes(prob, nb, xe.ModelOptions(strict_free=True), valid_mask=0)
    assert np.array_equal(r.obj.cpu().numpy().view(np.int64), o.view(np.int64))
    assert np.array_equal(r.flags.cpu().numpy().astype(np.uint32), f)


def test_move_placements_neighbours():
    # K4 placement moves: copies of the base with <= max_moves ops moved, only
    # to devices that can run them (fig2: op 0 never on the gpu), deterministic
    prob = xe.Problem.from_json(golden_problem_text("fig2"))
    cost = prob.arrays()["cost_ms"]
    base = torch.tensor([[0, 1, 1, 1, 1, 1, 0], [0, 0, 0, 0, 0, 0, 0]], dtype=torch.uint8, device="cuda")
    nb = xe.move_placements(prob, base, 2 * 4096, seed=5, max_moves=3)
    assert torch.equal(nb, xe.move_placements(prob, base, 2 * 4096, seed=5, max_moves=3))
    h = nb.cpu().numpy()
    b = base.cpu().numpy()
    diff = (h != np.repeat(b, 4096, axis=0)).sum(1)
    assert diff.max() <= 3 and (diff > 0).mean() > 0.5
    allowed = cost.T < 1e9  # [T, D]
    assert allowed[np.arange(prob.T)[None, :], h].all()
    assert (h[:, 0] == 0).all()


@pytest.mark.parametrize("name", ["fig2", "vgg16"])
def test_batched_rounding_equals_warp_rounding(name):
    # round_batch_kernel (one lane per candidate for the edits) and round_kernel
    # (lane 0 per candidate) run the same Philox streams and edit code
    import os
    text = golden_problem_text(name) if name == "fig2" else configs.CONFIGS[name]()
    prob = xe.Problem.from_json(text)
    a = xe.round_cubes(prob, 3000, seed=13, first=77, edits=4, perturb=0.2)
    os.environ["XE_ROUND_BATCH"] = "0"  # the warp-per-candidate kernel
    try:
        b = xe.round_cubes(prob, 3000, seed=13, first=77, edits=4, perturb=0.2)
    finally:
        del os.environ["XE_ROUND_BATCH"]
    assert torch.equal(a, b)


@pytest.mark.parametrize("name,edits", [("fig2", 6), ("vgg16", 4), ("resnet50", 5)])
@pytest.mark.parametrize("batch", ["6", "0"])
def test_fast_consumer_lookup_equals_row_scan(name, edits, batch, monkeypatch):
    # the edits' "latest step before t computing a consumer of u" from the
    # consumer rows + the candidate's own recomputation steps (default) and
    # from the backward scan over every step's R rows (XE_ROUND_SLOW_SCAN=1),
    # in both rounding kernels; and both minimal-save builds (word by word /
    # one atomic per saved bit, XE_ROUND_WORD) give the same cubes
    text = golden_problem_text(name) if name == "fig2" else configs.CONFIGS[name]()
    prob = xe.Problem.from_json(text)
    monkeypatch.setenv("XE_ROUND_BATCH", batch)
    n = 2000 if name != "resnet50" else 300
    a = xe.round_cubes(prob, n, seed=5, first=3, edits=edits, perturb=0.1)
    monkeypatch.setenv("XE_ROUND_SLOW_SCAN", "1")
    b = xe.round_cubes(prob, n, seed=5, first=3, edits=edits, perturb=0.1)
    assert torch.equal(a, b)
    monkeypatch.delenv("XE_ROUND_SLOW_SCAN")
    for w in ("0", "1"):
        monkeypatch.setenv("XE_ROUND_WORD", w)
        assert torch.equal(xe.round_cubes(prob, n, seed=5, first=3, edits=edits, perturb=0.1), a)
