# SPDX-License-Identifier: Apache-2.0
"""K2b's bit-sliced save-all kernel (eval_place.cu place_sliced_kernel)
against the warp-per-placement kernel (XE_PLACE_SLICED=0), whose outputs the
reference goldens pin (tests/test_place_gpu.py): every objective bit, peak
and flag equal, for 1..8 devices (1..3 bit planes), operator counts on and
off the 16-op vector blocks, and batches that end in a partial group of 32."""
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2212_09290_b200 as xe  # noqa: E402
from bench import configs  # noqa: E402


@pytest.mark.parametrize("D,T,n", [(2, 37, 1000), (3, 64, 777), (5, 130, 2049), (8, 208, 513), (8, 2000, 96)])
def test_sliced_equals_warp_kernel(D, T, n, monkeypatch):
    devices = ["cpu"] + [f"gpu{k}" for k in range(D - 1)]
    doc = configs._random_costs_doc(f"rand{D}x{T}", T, configs.random_dag_edges(T, seed=T + D), devices, seed=D)
    p = xe.Problem.from_json(doc)
    dev = xe.random_placements(p, n, 11)
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("XE_PLACE_SLICED", mode)
        r = xe.evaluate_placements(p, dev, policy=0)
        torch.cuda.synchronize()
        res[mode] = (r.obj.view(torch.int64).clone(), r.peak.clone(), r.flags.clone(), r.best_obj, r.best_index,
                     r.n_valid)
    a, b = res["1"], res["0"]
    assert torch.equal(a[0], b[0])
    assert torch.equal(a[1], b[1])
    assert torch.equal(a[2], b[2])
    assert a[3:] == b[3:]
