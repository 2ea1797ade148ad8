# SPDX-License-Identifier: Apache-2.0
"""K1 parity on the GPU: the device-assembled model equals the reference's
build_model (through the oracle's restatement, itself pinned to the
reference) array for array, and xe_write_mps reproduces the reference's MPS
bytes (golden f1 file and sha256 of the reference output for fixtures x
options, VGG-16 and ResNet-50)."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import FIXTURES, GOLDEN, golden_problem_text
from oracle import xo
from bench import configs

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2212_09290_b200 as xe  # noqa: E402


def text_of(name):
    if name in FIXTURES:
        return golden_problem_text(name)
    if name.startswith("rand"):
        return configs.random_small_doc(int(name[4:]))
    return configs.CONFIGS[name]()


def test_f1_golden_bytes():
    m = xe.build_model(xe.Problem.from_json(text_of("chain3")))
    with open(os.path.join(GOLDEN, "f1_golden.mps"), "rb") as f:
        assert m.write_mps() == f.read()


def test_mps_sha_against_reference():
    table = json.load(open(os.path.join(GOLDEN, "mps_sha256.json")))
    probs = {}
    for key, want in sorted(table.items()):
        name, opt = key.split("/")
        strict, quad, en = int(opt[1]), int(opt[3]), int(opt[5])
        if name not in probs:
            probs[name] = xe.Problem.from_json(text_of(name))
        m = xe.build_model(probs[name], xe.ModelOptions(strict_free=bool(strict),
                                                         quadratic_objective=bool(quad), energy=bool(en)))
        text = m.write_mps()
        assert len(text) == want["len"], key
        assert hashlib.sha256(text).hexdigest() == want["sha256"], key


@pytest.mark.parametrize("name", FIXTURES + ["vgg16", "rand3"])
@pytest.mark.parametrize("strict", [False, True])
def test_csr_arrays_equal_oracle(oracle, name, strict):
    text = text_of(name)
    a = xo.arrays_from_json(text)
    energies = (False, True) if a.energy is not None else (False,)
    prob = xe.Problem.from_json(text)
    for en in energies:
        want = oracle.build_model(a, strict, en)
        m = xe.build_model(prob, xe.ModelOptions(strict_free=strict, energy=en))
        got = m.to_host()
        assert (m.n_rows, m.nnz, m.n_cols) == (want.n_rows, want.nnz, want.n_cols)
        for k in ("row_ptr", "col", "val", "rhs", "sense", "tag", "ordinal"):
            assert np.array_equal(got[k], getattr(want, k)), k
        assert np.array_equal(got["obj"], want.obj)
        assert np.array_equal(got["obj_present"], want.obj_present)
        assert np.array_equal(got["kind"] == 0, want.fixed.astype(bool))


def test_csc_is_stable_transpose(oracle):
    prob = xe.Problem.from_json(text_of("fig2"))
    m = xe.build_model(prob)
    h = m.to_host()
    c = {k: v.cpu().numpy() for k, v in m.csc().items()}
    rows = np.repeat(np.arange(m.n_rows), np.diff(h["row_ptr"]))
    order = np.lexsort((rows, h["col"]))
    assert np.array_equal(c["row"], rows[order])
    assert np.array_equal(c["val"], h["val"][order])
    assert np.array_equal(c["col_ptr"], np.searchsorted(h["col"][order], np.arange(m.n_cols + 1)))


def test_config3_shape_and_timing():
    # ResNet-50 cfg3: 1,015,581 rows, 4,348,851 nnz, 659,895 columns
    prob = xe.Problem.from_json(configs.resnet50_doc())
    m = xe.build_model(prob)
    assert (m.n_rows, m.nnz, m.n_cols) == (1015581, 4348851, 659895)
    assert m.build_ms() > 0


def _fractional_energy_doc(seed):
    """fig2_energy with every number made non-integral: the device writer's
    host-formatted number table must cover costs, copy costs, alpha*q, the
    energy coefficients and limits."""
    rng = np.random.default_rng(seed)
    d = json.loads(golden_problem_text("fig2_energy"))
    for op in d["operators"][1:]:
        op["costs_ms"] = {k: float(v * rng.uniform(0.3, 3.0) + 0.1) for k, v in op["costs_ms"].items()}
    for e in d["edges"]:
        e["copy_ms"] = {k: float(v * rng.uniform(0.1, 2.0)) for k, v in e["copy_ms"].items()}
    en = d["energy"]
    en["alpha"] = float(rng.uniform(0.01, 2.0))
    en["q_joules"] = {k: [float(x * rng.uniform(0.1, 3.0)) for x in v] for k, v in en["q_joules"].items()}
    en["board_joules"] = float(rng.uniform(0.0, 2.0))
    en["device_limit"] = {"gpu": float(rng.uniform(4.0, 9.0)), "cpu": float(rng.uniform(4.0, 9.0))}
    en["total_limit"] = float(rng.uniform(10.0, 20.0))
    return json.dumps(d)


@pytest.mark.parametrize("seed", range(4))
def test_device_mps_equals_host_writer(seed, monkeypatch):
    """xe_write_mps's device emitter (mps_device.cu) and the host writer
    (mps_writer.cpp) agree byte for byte on fractional energy models (the
    sha table above covers integral ones and ResNet-50/U-Net)."""
    prob = xe.Problem.from_json(_fractional_energy_doc(seed))
    for strict in (False, True):
        for quad in (False, True):
            opts = xe.ModelOptions(strict_free=strict, quadratic_objective=quad, energy=True)
            monkeypatch.delenv("XE_MPS_HOST", raising=False)
            dev = xe.build_model(prob, opts).write_mps()
            monkeypatch.setenv("XE_MPS_HOST", "1")
            host = xe.build_model(prob, opts).write_mps()
            assert dev == host, (seed, strict, quad)
            assert b"ENERGY_TOTAL" in dev
