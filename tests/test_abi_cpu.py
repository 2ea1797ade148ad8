# SPDX-License-Identifier: Apache-2.0
"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/xengine_b200.h declares, maps errors like the reference, and
the host loader reproduces the reference loader (proj/src/problem.cpp)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import FIXTURES, ROOT, golden_problem_text
from oracle import xo
from bench import configs

import paper_2212_09290_b200 as xe
from paper_2212_09290_b200 import _lib


def header_functions():
    text = open(os.path.join(ROOT, "include", "xengine_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(xe_[a-z_0-9]+)\s*\(", text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 20
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a():
    # the shared object carries sm_100a SASS (no PTX-only / other-arch fallback)
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def parse(text):
    h = C.c_void_p()
    st = _lib.LIB.xe_problem_parse_json(text.encode(), C.byref(h))
    if st != 0:
        raise _lib.XeError(st, _lib.LIB.xe_last_error().decode())
    d = _lib.ProblemDesc()
    _lib.check(_lib.LIB.xe_problem_describe(h, C.byref(d)))

    def arr(ptr, n, dt):
        if n == 0:
            return np.zeros(0, dt)
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), shape=(n,)).copy()

    D, T, E = d.D, d.T, d.E
    out = dict(D=D, T=T, E=E, mass=arr(d.output_bytes, T, np.int64),
               cost=arr(d.cost_ms, D * T, np.float64).reshape(D, T),
               src=arr(d.edge_src, E, np.int32), dst=arr(d.edge_dst, E, np.int32),
               w=arr(d.copy_ms, E * D * D, np.float64).reshape(E, D, D),
               budget=arr(d.budget_bytes, D, np.int64), has_energy=d.has_energy,
               q=arr(d.q_joules, D * T, np.float64).reshape(D, T),
               has_lim=arr(d.has_dev_limit, D, np.uint8), lim=arr(d.dev_limit, D, np.float64))
    _lib.LIB.xe_problem_destroy(h)
    return out


DOCS = {**{n: (lambda n=n: golden_problem_text(n)) for n in FIXTURES},
        "fig2_layered": configs.fig2_doc, "vgg16": configs.vgg16_doc,
        "resnet50": configs.resnet50_doc, "unet": configs.unet_doc,
        "random2000": configs.random2000_doc,
        "rand3": lambda: configs.random_small_doc(3)}


@pytest.mark.parametrize("name", sorted(DOCS))
def test_loader_matches_reference_restatement(name):
    text = DOCS[name]()
    got = parse(text)
    want = xo.arrays_from_json(text)
    for k in ("mass", "cost", "src", "dst", "w", "budget"):
        assert np.array_equal(got[k], getattr(want, k)), k
    assert bool(got["has_energy"]) == (want.energy is not None)
    if want.energy is not None:
        assert np.array_equal(got["q"], want.q)
        assert np.array_equal(got["has_lim"], want.has_lim)
        assert np.array_equal(got["lim"], want.lim)


@pytest.mark.skipif(not xo.ref_available(), reason="reference library not built here")
@pytest.mark.parametrize("name", sorted(DOCS))
def test_loader_matches_compiled_reference(name):
    text = DOCS[name]()
    got = parse(text)
    want = xo.Ref().load(text).arrays()
    for k in ("mass", "cost", "src", "dst", "w", "budget"):
        assert np.array_equal(got[k], getattr(want, k)), k


BAD = {
    "MalformedDocument": ['{"devices": []}', "not json", "[]",
                          '{"devices":[{"id":"a","budget_bytes":1}],"operators":[{"name":"x","output_bytes":1,"costs_ms":{}},'
                          '{"name":"y","output_bytes":1,"costs_ms":{}}],"edges":[]}'],
    "NonTopologicalEdge": ['{"devices":[{"id":"a","budget_bytes":1}],"operators":[{"name":"x","output_bytes":1,"costs_ms":{}},'
                           '{"name":"y","output_bytes":1,"costs_ms":{}}],"edges":[[1,0]]}'],
    "UnknownDevice": ['{"devices":[{"id":"a","budget_bytes":1}],"operators":[{"name":"x","output_bytes":1,"costs_ms":{"b":1}}]}'],
    "NonPositiveSize": ['{"devices":[{"id":"a","budget_bytes":0}],"operators":[{"name":"x","output_bytes":1,"costs_ms":{}}]}'],
    "NegativeCost": ['{"devices":[{"id":"a","budget_bytes":1}],"operators":[{"name":"x","output_bytes":1,"costs_ms":{"a":-1}}]}'],
    "EmptyNetwork": ['{"devices":[{"id":"a","budget_bytes":1}],"operators":[]}'],
}


@pytest.mark.parametrize("code", sorted(BAD))
def test_loader_error_codes(code):
    # proj/tests/test_problem.cpp: loader errors carry the reference's Errc
    for text in BAD[code]:
        with pytest.raises(_lib.XeError) as ei:
            parse(text)
        assert ei.value.code == code, (text, ei.value)
        with pytest.raises(xo.OracleError) as eo:
            xo.load_problem(text)
        assert eo.value.code == code


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.XeError) as ei:
        xe.Problem.from_json(golden_problem_text("fig2"))
    assert ei.value.code == "NoDevice"


def test_search_abi_defaults_and_argument_checks():
    """xe_search_opts_default fills the documented defaults; xe_search
    rejects a null problem before touching a device."""
    import ctypes as C
    o = _lib.SearchOpts()
    _lib.LIB.xe_search_opts_default(C.byref(o))
    assert (o.n_per_round, o.rounds, o.edits, o.seed, o.use_lp) == (1 << 18, 4, 3, 1, 1)
    assert o.valid_mask == (_lib.F_CHECK_MASK | _lib.F_BUDGET | _lib.F_DECODE)
    assert (o.canonical, o.chains, o.chain_n, o.chain_iters, o.max_moves, o.stall) == (1, 256, 1024, 200, 4, 15)
    assert (o.first, o.rank, o.world, o.time_limit_ms) == (0, 0, 1, 0)
    r = _lib.SearchResult()
    rc = _lib.LIB.xe_search(None, None, C.byref(o), C.byref(r), None, None, None)
    assert rc == 102  # XE_ERR_ARG
