# SPDX-License-Identifier: Apache-2.0
"""The N>1 path on CPU: world_size-2 gloo process groups run the sharding and
the incumbent exchange (paper_2212_09290_b200/shard.py) on per-rank bests
computed by the CPU oracle, and must reproduce the single-process first
minimum (solver.cpp:57-61 tie rule) over the concatenated candidates."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2212_09290_b200.shard import exchange_best, shard_range


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def first_min(obj, valid):
    idx = np.nonzero(valid)[0]
    if len(idx) == 0:
        return float("inf"), -1
    k = idx[np.argmin(obj[idx])]
    return float(obj[k]), int(k)


def _worker(rank, world, port, case, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        obj, valid = case
        lo, hi = shard_range(len(obj), rank, world)
        o, i = first_min(obj[lo:hi], valid[lo:hi])
        inc = exchange_best(o, i, int(valid[lo:hi].sum()), offset=lo, device="cpu")
        q.put((rank, inc.obj, inc.index, inc.n_valid))
    finally:
        dist.destroy_process_group()


def run_world(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return out


def test_shard_range_partitions():
    for n in (0, 1, 7, 32, 1001):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1


@pytest.mark.parametrize("kind", ["random", "tie_across_ranks", "one_rank_empty", "none_valid"])
def test_exchange_matches_single_process(kind):
    rng = np.random.default_rng(3)
    n = 200
    obj = rng.integers(10, 50, n).astype(np.float64) * 0.25
    valid = rng.random(n) < 0.6
    if kind == "tie_across_ranks":
        obj[:] = 40.0
        obj[150] = obj[30] = 3.0  # equal minima on both ranks: the lower index wins
        valid[150] = valid[30] = True
    if kind == "one_rank_empty":
        valid[:100] = False
    if kind == "none_valid":
        valid[:] = False
    want_obj, want_idx = first_min(obj, valid)
    for rank, o, i, nv in run_world((obj, valid)):
        assert i == want_idx and nv == int(valid.sum())
        assert (o == want_obj) or (want_idx < 0 and o == float("inf"))


def test_sharded_oracle_sweep_matches_full(oracle):
    """K2 semantics sharded over 2 ranks: oracle-evaluated VGG-16 candidates."""
    from bench import configs
    from oracle import xo
    import cubegen
    text = configs.vgg16_doc()
    a = xo.arrays_from_json(text)
    cubes = cubegen.mixed_cubes(a, 96, seed=11, random_frac=0.1)
    o, p, f = oracle.eval_cubes(a, cubes)
    valid = (f & 0x7FFF) == 0
    want_obj, want_idx = first_min(o, valid)
    for rank, go, gi, nv in run_world((o, valid)):
        assert gi == want_idx and go == want_obj and nv == int(valid.sum())
