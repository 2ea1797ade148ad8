# SPDX-License-Identifier: Apache-2.0
"""Pins the CPU oracle (oracle/xe_oracle.c + oracle/xo.py) to the reference:
its own golden MPS file, fixture pins from proj/tests, and golden vectors
produced by the compiled reference (scripts/gen_golden.py).  CPU only."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import FIXTURES, GOLDEN, golden_npz, golden_problem_text, pins
from oracle import xo
from bench import configs


def arrays(name):
    return xo.arrays_from_json(golden_problem_text(name))


def test_format_number_reference_cases(oracle):
    # proj/tests/test_mps_io.cpp:85-99
    cases = {0.0: "0", 1.0: "1", -3.0: "-3", 2.5: "2.5", 0.1: "0.1", 1e9: "1000000000",
             12582912.0: "12582912", 1.0 / 3.0: "0.3333333333333333"}
    for v, s in cases.items():
        assert oracle.format_number(v) == s
    for v in (0.1, 1.0 / 3.0, 1e-9, 123456.789, 0.25, 2.0 / 7.0):
        assert float(oracle.format_number(v)) == v


def test_f1_golden_mps_bytes(oracle):
    # proj/tests/test_mps_io.cpp:120-124: chain3 MPS equals the golden file
    with open(os.path.join(GOLDEN, "f1_golden.mps"), "rb") as f:
        assert oracle.write_mps(arrays("chain3")) == f.read()


def test_mps_sha_fixtures_and_configs(oracle):
    table = json.load(open(os.path.join(GOLDEN, "mps_sha256.json")))
    checked = 0
    for key, want in table.items():
        name, opt = key.split("/")
        strict, quad, en = int(opt[1]), int(opt[3]), int(opt[5])
        if name in FIXTURES:
            a = arrays(name)
        elif name == "vgg16":
            a = xo.arrays_from_json(configs.vgg16_doc())
        elif name.startswith("rand"):
            a = xo.arrays_from_json(configs.random_small_doc(int(name[4:])))
        else:
            continue  # resnet50 (196 MB) is checked on the GPU side
        text = oracle.write_mps(a, strict, quad, en)
        assert len(text) == want["len"], key
        assert hashlib.sha256(text).hexdigest() == want["sha256"], key
        checked += 1
    assert checked >= 40


def test_model_census_reference_pins(oracle):
    # proj/tests/test_model.cpp:39-90 (row census per tag; objective entries)
    tags = ["EQ7", "EQ8", "EQ9", "EQ10", "EQ11", "EQ12", "EQ13", "EQ14", "EQ16_LO", "EQ16_HI",
            "Z_LINK", "P_LINK", "ENERGY_DEV", "ENERGY_TOTAL"]
    m = oracle.build_model(arrays("chain3"))
    n = {t: int((m.tag == i).sum()) for i, t in enumerate(tags)}
    assert n["EQ8"] == 6 and n["EQ9"] == 1 and n["EQ11"] == 6 and n["EQ12"] == 6
    assert n["EQ13"] == 3 and n["EQ14"] == 6 and n["EQ16_LO"] == 15 and n["EQ16_HI"] == 15
    assert n["Z_LINK"] == 27 and n["P_LINK"] == 0
    assert int(m.obj_present.sum()) == 9 and int(m.fixed.sum()) == 9
    m2 = oracle.build_model(arrays("fig2"))
    assert int((m2.tag == 11).sum()) == 7 * 9 * 2
    assert int(m2.obj_present.sum()) == 98 - 7 + 126
    assert int(m2.fixed.sum()) == 2 * (21 + 28)
    # energy rows (test_model.cpp:189-270): 49 device rows for the gpu cap
    me = oracle.build_model(arrays("fig2_energy"), energy=True)
    assert int((me.tag == 12).sum()) == 49


def test_config_shapes_match_survey(oracle):
    # SURVEY §8 table (checked there against the reference's build_model)
    a = xo.arrays_from_json(configs.fig2_doc())
    m = oracle.build_model(a)
    assert (m.n_cols, m.n_rows, m.nnz) == (742, 1191, 4612)
    a = xo.arrays_from_json(configs.vgg16_doc())
    m = oracle.build_model(a)
    assert (a.T, a.E, m.n_cols, m.n_rows, m.nnz) == (43, 63, 29326, 47559, 190840)


@pytest.mark.parametrize("name", FIXTURES + ["vgg16", "rand3", "rand7", "rand11"])
def test_eval_matches_reference_golden(oracle, name):
    z = golden_npz("eval_" + name)
    if name in FIXTURES:
        a = arrays(name)
    elif name == "vgg16":
        a = xo.arrays_from_json(configs.vgg16_doc())
    else:
        a = xo.arrays_from_json(configs.random_small_doc(int(name[4:]), D=3))
    cubes = z["cubes"]
    if name == "vgg16":
        cubes = cubes[:120]  # the C oracle is O(nnz) per candidate
    for strict in (0, 1):
        for en in ((0, 1) if name == "fig2_energy" else (0,)):
            o, p, f = oracle.eval_cubes(a, cubes, strict, en)
            n = len(cubes)
            ro, rp, rf = z[f"obj_s{strict}e{en}"][:n], z[f"peak_s{strict}e{en}"][:n], z[f"flags_s{strict}e{en}"][:n]
            assert np.array_equal(o.view(np.int64), ro.view(np.int64)), "objective bits"
            assert np.array_equal(p, rp)
            mask = 0xFFFF | xo.F_DECODE
            assert np.array_equal(f & mask, rf & mask)
            # DECODE_FREED: the reference reports the first decode error only;
            # it is comparable wherever no dependency is resident nowhere
            comparable = (rf & xo.F_DECODE) != 0
            comparable &= (f & xo.F_EQ12) == 0
            assert np.array_equal((f & xo.F_DECODE_FREED)[comparable], (rf & xo.F_DECODE_FREED)[comparable])


@pytest.mark.parametrize("name", ["fig2", "vgg16"])
def test_placements_match_reference_golden(oracle, name):
    z = golden_npz("place_" + name)
    a = arrays(name) if name == "fig2" else xo.arrays_from_json(configs.vgg16_doc())
    dev = z["dev"][:100]
    for pol in (0, 1):
        o, p, f = oracle.eval_placements(a, dev, pol)
        assert np.array_equal(o.view(np.int64), z[f"obj_p{pol}"][:100].view(np.int64))
        assert np.array_equal(p, z[f"peak_p{pol}"][:100])
        assert np.array_equal(f & 0xFFFF, z[f"flags_p{pol}"][:100] & 0xFFFF)


def test_assignment_oracle_pins(oracle):
    pn = pins()
    # proj/tests/test_solver.cpp:99-119: fig2 oracle = 11.0
    o, dev, n = oracle.assignment_oracle(arrays("fig2"))
    assert o == pn["fig2/oracle"]["obj"] == 11.0
    assert dev.tolist() == pn["fig2/oracle"]["dev"]
    assert n == 2 ** 7
    for seed in (1, 2, 3):
        a = xo.arrays_from_json(configs.random_small_doc(seed))
        o, dev, _ = oracle.assignment_oracle(a)
        assert o == pn[f"rand{seed}"]["oracle"]
        assert dev.tolist() == pn[f"rand{seed}"]["oracle_dev"]


def test_reference_pins_values():
    pn = pins()
    assert pn["chain3/exact"]["obj"] == 9.0          # test_solver.cpp:66-86
    assert pn["fig2/exact"]["obj"] == 11.0           # test_solver.cpp:99-119
    sweep = [pn[f"chain_lowmem/exact@{p}"]["obj"] for p in (100, 65, 50, 35, 25)]
    assert sweep == [24.0, 24.0, 24.0, 24.0, 27.0]   # test_solver.cpp:121-153
    assert pn["fig2_energy/exact"]["obj"] == 11.0 or pn["fig2_energy/exact"]["status"] in (0, 1)


def test_loader_restatement_matches_reference_arrays():
    # the Python restatement of problem.cpp reproduces the golden documents' arrays
    for name in FIXTURES:
        a = arrays(name)
        assert a.T > 0 and a.w.shape == (a.E, a.D, a.D)
    assert xo.budget_percent(320 * 1048576, 65.0) == 208 * 1048576   # test_problem.cpp:121-126
    assert xo.budget_percent(100, 100.0) == 100
    assert xo.budget_percent(101, 50.0) == 50
    for bad in (0.0, 100.5):
        with pytest.raises(xo.OracleError):
            xo.budget_percent(100, bad)
