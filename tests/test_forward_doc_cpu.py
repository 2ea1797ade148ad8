# SPDX-License-Identifier: Apache-2.0
"""Forward-DAG training documents (the loader's "forward" form,
csrc/loader.cpp expand_training_graph — make_training_graph,
proj/src/problem.cpp:280-338, generalised from a layer chain to a forward
DAG).  Host-only parse through the C ABI (no device)."""
import ctypes as C
import json

import numpy as np
import pytest

from bench import configs
from paper_2212_09290_b200 import _lib


def arrays(text):
    h = C.c_void_p()
    _lib.check(_lib.LIB.xe_problem_parse_json(text.encode(), C.byref(h)))
    d = _lib.ProblemDesc()
    _lib.check(_lib.LIB.xe_problem_describe(h, C.byref(d)))
    D, T, E = d.D, d.T, d.E
    def arr(ptr, ct, n):
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), (n,)).copy() if n else np.zeros(0)
    out = {"D": D, "T": T, "E": E,
           "mass": arr(d.output_bytes, C.c_int64, T), "cost": arr(d.cost_ms, C.c_double, D * T),
           "src": arr(d.edge_src, C.c_int32, E), "dst": arr(d.edge_dst, C.c_int32, E),
           "w": arr(d.copy_ms, C.c_double, E * D * D), "budget": arr(d.budget_bytes, C.c_int64, D)}
    _lib.LIB.xe_problem_destroy(h)
    return out


def chain_forward_doc(layered_text):
    d = json.loads(layered_text)
    fwd = []
    for k, l in enumerate(d["layers"]):
        fwd.append(dict(l, inputs=[k]))
    d["forward"] = fwd
    del d["layers"]
    return json.dumps(d)


def test_chain_forward_equals_layered_vgg16():
    # a chain in the forward form is the reference's make_training_graph exactly:
    # same operators, same edge order (forward chain, then gradient + saved per backward op)
    a = arrays(configs.vgg16_doc())
    b = arrays(chain_forward_doc(configs.vgg16_doc()))
    for k in a:
        assert np.array_equal(a[k], b[k]) if isinstance(a[k], np.ndarray) else a[k] == b[k], k


def test_chain_forward_equals_reference_training_graph():
    from oracle import xo
    if not xo.ref_available():
        pytest.skip("oracle/_ref not built")
    ref = xo.Ref().load(configs.vgg16_doc()).arrays()
    b = arrays(chain_forward_doc(configs.vgg16_doc()))
    assert np.array_equal(ref.src, b["src"]) and np.array_equal(ref.dst, b["dst"])
    assert np.array_equal(ref.mass, b["mass"])
    assert np.array_equal(ref.cost.ravel(), b["cost"])


@pytest.mark.parametrize("name", ["resnet50", "unet"])
def test_dag_forward_doc_expands_to_the_config(name):
    # configs 3/4 written as forward networks: the expansion has exactly the
    # direct document's operators and edge set (the direct form sorts its edges)
    direct = arrays(configs.CONFIGS[name]())
    fdoc = {"resnet50": configs.resnet50_forward_doc, "unet": configs.unet_forward_doc}[name]()
    got = arrays(fdoc)
    assert (got["D"], got["T"], got["E"]) == (direct["D"], direct["T"], direct["E"])
    assert np.array_equal(got["mass"], direct["mass"]) and np.array_equal(got["cost"], direct["cost"])
    assert set(zip(got["src"].tolist(), got["dst"].tolist())) == set(zip(direct["src"].tolist(),
                                                                          direct["dst"].tolist()))


def test_forward_doc_errors():
    d = json.loads(chain_forward_doc(configs.vgg16_doc()))
    d["forward"][3]["inputs"] = [7]  # not an earlier op
    with pytest.raises(_lib.XeError) as ei:
        arrays(json.dumps(d))
    assert ei.value.code == "NonTopologicalEdge"
    d["forward"][3]["inputs"] = []
    with pytest.raises(_lib.XeError) as ei:
        arrays(json.dumps(d))
    assert ei.value.code == "MalformedDocument"
