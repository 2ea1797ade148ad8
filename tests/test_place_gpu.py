# SPDX-License-Identifier: Apache-2.0
"""K2b placements and the GPU assignment oracle against the reference
(golden vectors from save_all_assignment + objective_value/check_assignment,
and solve pins) and against the CPU oracle."""
import numpy as np
import pytest

from conftest import golden_npz, golden_problem_text, pins
from oracle import xo
from bench import configs
import cubegen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200 import _lib  # noqa: E402
import ctypes as C  # noqa: E402


def place(prob, dev, policy):
    n = dev.shape[0]
    d = torch.from_numpy(np.ascontiguousarray(dev, np.uint8)).cuda()
    obj = torch.empty(n, dtype=torch.float64, device="cuda")
    pk = torch.empty((n, prob.D), dtype=torch.int64, device="cuda")
    fl = torch.empty(n, dtype=torch.int32, device="cuda")
    out = _lib.EvalOut(C.c_void_p(obj.data_ptr()), C.c_void_p(pk.data_ptr()), C.c_void_p(fl.data_ptr()))
    best = _lib.Best()
    _lib.check(_lib.LIB.xe_eval_placements(prob.handle, C.c_void_p(d.data_ptr()), n, policy, C.byref(out),
                                           _lib.F_CHECK_MASK, C.byref(best), None))
    torch.cuda.synchronize()
    return obj.cpu().numpy(), pk.cpu().numpy(), fl.cpu().numpy().view(np.uint32), best


@pytest.mark.parametrize("name", ["fig2", "vgg16"])
def test_placements_vs_reference_golden(name):
    z = golden_npz("place_" + name)
    text = golden_problem_text("fig2") if name == "fig2" else configs.vgg16_doc()
    prob = xe.Problem.from_json(text)
    for pol in (0, 1):
        o, p, f, _ = place(prob, z["dev"], pol)
        assert np.array_equal(o.view(np.int64), z[f"obj_p{pol}"].view(np.int64))
        assert np.array_equal(p, z[f"peak_p{pol}"])
        assert np.array_equal(f & 0xFFFF, z[f"flags_p{pol}"] & 0xFFFF)


@pytest.mark.parametrize("name", ["resnet50", "unet"])
def test_placements_vs_oracle_large(oracle, name):
    text = configs.CONFIGS[name]()
    a = xo.arrays_from_json(text)
    prob = xe.Problem.from_json(text)
    dev = cubegen.random_placements(a, 40, np.random.default_rng(1))
    for pol in (0, 1):
        o, p, f, _ = place(prob, dev, pol)
        ro, rp, rf = oracle.eval_placements(a, dev, pol)
        assert np.array_equal(o.view(np.int64), ro.view(np.int64))
        assert np.array_equal(p, rp)
        assert np.array_equal(f & 0xFFFF, rf & 0xFFFF)


def test_placements_equal_cube_path():
    # a placement and its cube evaluate identically through K2a and K2b
    text = configs.vgg16_doc()
    a = xo.arrays_from_json(text)
    prob = xe.Problem.from_json(text).set_exact_objective()  # K2b sums in the reference's order
    dev = cubegen.random_placements(a, 500, np.random.default_rng(3))
    for pol in (0, 1):
        o, p, f, _ = place(prob, dev, pol)
        Rb, Sb = cubegen.placement_cubes(a, dev.astype(np.int64), policy=pol)
        cubes = cubegen.pack(Rb, Sb)
        r = xe.evaluate_cubes(prob, torch.from_numpy(cubes.view(np.int32)).cuda())
        assert np.array_equal(r.obj.cpu().numpy().view(np.int64), o.view(np.int64))
        assert np.array_equal(r.peak.cpu().numpy(), p)


def test_random2000_placements_run():
    prob = xe.Problem.from_json(configs.random2000_doc())
    dev = np.random.default_rng(0).integers(0, 8, size=(64, 2000)).astype(np.uint8)
    dev[:, 0] = 0
    o, p, f, best = place(prob, dev, 0)
    assert np.isfinite(o).all() and (p.sum(1) == prob.arrays()["output_bytes"].sum()).all()


def _oracle(prob):
    obj = C.c_double()
    dev = np.zeros(prob.T, np.int32)
    n = C.c_int64()
    _lib.check(_lib.LIB.xe_assignment_oracle(prob.handle, C.byref(obj), dev.ctypes.data, C.byref(n)))
    return obj.value, dev, n.value


def test_assignment_oracle_pins():
    pn = pins()
    o, dev, n = _oracle(xe.Problem.from_json(golden_problem_text("fig2")))
    assert o == pn["fig2/oracle"]["obj"] == 11.0 and dev.tolist() == pn["fig2/oracle"]["dev"] and n == 128
    for seed in range(1, 21):
        o, dev, _ = _oracle(xe.Problem.from_json(configs.random_small_doc(seed)))
        assert o == pn[f"rand{seed}"]["oracle"]
        assert dev.tolist() == pn[f"rand{seed}"]["oracle_dev"]
        assert pn[f"rand{seed}"]["exact"] <= o + 1e-9  # oracle dominance (test_properties.cpp:71-75)


@pytest.mark.parametrize("name", ["fig2", "random2000"])
def test_random_placements_generator_and_api(oracle, name):
    """K4-style placement generator (config 5's sweep input): index-deterministic,
    never on a prohibitive device; the Python API agrees with the CPU oracle."""
    text = golden_problem_text("fig2") if name == "fig2" else configs.random2000_doc()
    a = xo.arrays_from_json(text)
    prob = xe.Problem.from_json(text)
    n = 4000 if name == "fig2" else 48
    dev = xe.random_placements(prob, n, seed=9)
    parts = torch.cat([xe.random_placements(prob, n // 2, seed=9), xe.random_placements(prob, n - n // 2, seed=9, first=n // 2)])
    assert torch.equal(dev, parts)
    dv = dev.cpu().numpy()
    cost = np.asarray(a.cost).reshape(a.D, a.T)
    assert (cost[dv, np.arange(a.T)[None, :]] < 1e9).all()
    assert len(np.unique(dv[:, 1:])) == a.D
    if name == "fig2":
        for pol in (0, 1):
            r = xe.evaluate_placements(prob, dev, policy=pol)
            ro, rp, rf = oracle.eval_placements(a, dv, pol)
            assert np.array_equal(r.obj.cpu().numpy().view(np.int64), ro.view(np.int64))
            assert np.array_equal(r.peak.cpu().numpy(), rp)
            assert np.array_equal(r.flags.cpu().numpy().view(np.uint32) & 0xFFFF, rf & 0xFFFF)
    else:
        # T = 2000: the dense oracle is out of reach (926 M columns); the
        # save-all closed forms with dyadic costs are exact in
        # any summation order
        r = xe.evaluate_placements(prob, dev, policy=0)
        ar = np.arange(a.T)
        want = cost[dv, ar[None, :]].sum(axis=1) + np.where(
            dv[:, a.src] != dv[:, a.dst], a.w[np.arange(a.E)[None, :], dv[:, a.src], dv[:, a.dst]], 0.0).sum(axis=1)
        assert np.array_equal(r.obj.cpu().numpy(), want)
        peak = np.stack([(a.mass[None, :] * (dv == d)).sum(axis=1) for d in range(a.D)], axis=1)
        assert np.array_equal(r.peak.cpu().numpy(), peak)


def test_oracle_python_api_fig2():
    obj, dev, n = xe.assignment_oracle(xe.Problem.from_json(golden_problem_text("fig2")))
    assert obj == 11.0 and n == 128 and dev[1] == 0  # A on the cpu (test_solver.cpp:99-119)
