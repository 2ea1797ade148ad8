# SPDX-License-Identifier: Apache-2.0
"""Multi-GPU plumbing for the candidate sweeps (one process per GPU).

Candidates shard with no data-path collective: rank r owns the contiguous
global index range shard_range(n, r, world) (K4 candidates are pure functions
of (seed, global index), so a shard regenerates its own inputs).  The only
exchange is the incumbent: the global first minimum over valid candidates,
the multi-GPU form of the reference's first-strict-improvement rule
(proj/src/solver.cpp:57-61):

  1. all-reduce MIN of the objective's IEEE bits as int64 (objectives are
     non-negative, so their bit patterns order like the values; "no valid
     candidate" is INT64_MAX),
  2. all-reduce MIN of the global index over ranks holding that objective,
  3. all-reduce SUM of the valid counts.

Three 8-byte messages (NCCL over NVLink on the GPU box; gloo in the CPU tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

NONE = np.iinfo(np.int64).max


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of rank among world."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def objective_key(obj: float, index: int) -> int:
    """int64 key of a shard's best (NONE when the shard has no valid candidate)."""
    if index < 0:
        return NONE
    return int(np.float64(obj).view(np.int64))


@dataclass
class Incumbent:
    obj: float
    index: int      # global candidate index, -1 if none
    n_valid: int


def exchange_best(obj: float, index: int, n_valid: int, offset: int = 0, device=None, group=None) -> Incumbent:
    """Global first minimum of the per-rank bests (index local to the shard,
    offset = the shard's first global index)."""
    import torch
    import torch.distributed as dist
    dev = device if device is not None else ("cuda" if dist.get_backend(group) == "nccl" else "cpu")
    key = objective_key(obj, index)
    t = torch.tensor([key], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    gkey = int(t.item())
    gi = offset + index if (index >= 0 and key == gkey) else NONE
    t = torch.tensor([gi, n_valid], dtype=torch.int64, device=dev)
    u = t[:1].clone()
    dist.all_reduce(u, op=dist.ReduceOp.MIN, group=group)
    v = t[1:].clone()
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    if gkey == NONE:
        return Incumbent(float("inf"), -1, int(v.item()))
    return Incumbent(float(np.int64(gkey).view(np.float64)), int(u.item()), int(v.item()))


class NcclContext:
    """The native multi-GPU context of the C ABI (xe_ctx: device, rank, world,
    NCCL communicator; csrc/dist.cpp) for C/C++-style callers: rank 0 creates
    the NCCL id, which the caller distributes (here over torch.distributed
    when it is initialised).  exchange_best() and search() run the same
    exchanges as this module's torch.distributed versions, natively."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        import ctypes as C
        from . import _lib
        if nccl_id is None:
            buf = (C.c_uint8 * 128)()
            if rank == 0:
                _lib.check(_lib.LIB.xe_nccl_unique_id(buf))
            if world > 1:
                import torch
                import torch.distributed as dist
                t = torch.tensor(list(bytes(buf)), dtype=torch.uint8, device="cuda")
                dist.broadcast(t, src=0)
                buf = (C.c_uint8 * 128)(*t.cpu().tolist())
        else:
            buf = (C.c_uint8 * 128)(*nccl_id)
        self._h = C.c_void_p()
        _lib.check(_lib.LIB.xe_ctx_create(device, rank, world, buf, C.byref(self._h)))
        self.device, self.rank, self.world = device, rank, world

    def close(self):
        from . import _lib
        if self._h:
            _lib.check(_lib.LIB.xe_ctx_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def exchange_best(self, obj: float, index: int, n_valid: int, offset: int = 0) -> Incumbent:
        import ctypes as C
        from . import _lib
        b = _lib.Best(obj, index, n_valid)
        _lib.check(_lib.LIB.xe_ctx_exchange_best(self._h, offset, C.byref(b)))
        return Incumbent(b.obj, b.index, b.n_valid)

    def search(self, problem, opts=None, **kw):
        """xe_search_dist: the search sharded over this context's ranks."""
        import ctypes as C
        from . import _lib
        from .api import ModelOptions
        so = _lib.SearchOpts()
        _lib.LIB.xe_search_opts_default(C.byref(so))
        for k, v in kw.items():
            setattr(so, k, v)
        res = _lib.SearchResult()
        cube = np.zeros(problem.cube_words, np.uint32)
        peaks = np.zeros(problem.D, np.int64)
        mo = (opts or ModelOptions()).c()
        _lib.check(_lib.LIB.xe_search_dist(problem.handle, C.byref(mo), C.byref(so), self._h, C.byref(res),
                                           cube.ctypes.data, peaks.ctypes.data))
        return res, cube, peaks
