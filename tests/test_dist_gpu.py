# SPDX-License-Identifier: Apache-2.0
"""The native multi-GPU context of the C ABI (csrc/dist.cpp: xe_ctx with an
NCCL communicator).  The GPU box has one GPU, so the communicator is world 1
(NCCL refuses two ranks on one device); the exchange logic across ranks is
the same three-step rule tests/test_shard_cpu.py checks with gloo world 2."""
import numpy as np
import pytest

from conftest import golden_problem_text

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200.search import search  # noqa: E402
from paper_2212_09290_b200.shard import NcclContext  # noqa: E402


def test_ctx_exchange_world1():
    ctx = NcclContext(0, 0, 1)
    inc = ctx.exchange_best(12.5, 7, 100, offset=1000)
    assert (inc.obj, inc.index, inc.n_valid) == (12.5, 1007, 100)
    none = ctx.exchange_best(float("inf"), -1, 0)
    assert none.index == -1 and none.obj == float("inf")
    ctx.close()


def test_search_dist_world1_equals_search():
    p = xe.Problem.from_json(golden_problem_text("fig2"))
    ctx = NcclContext(0, 0, 1)
    res, cube, peaks = ctx.search(p, n_per_round=1 << 14, rounds=2, chains=16, chain_n=64, chain_iters=5)
    ref = search(p, n_per_round=1 << 14, rounds=2, chains=16, chain_n=64, chain_iters=5)
    assert res.objective == ref.objective == 11.0
    assert np.array_equal(cube, ref.cube) and peaks.tolist() == ref.peaks.tolist()
    ctx.close()
