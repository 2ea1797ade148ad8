# SPDX-License-Identifier: Apache-2.0
"""LP-guided randomised search for the best schedule (K1 -> K3 -> K4 -> K2).

The reference finds schedules with its exact memoised DFS (solve_exact,
proj/src/solver.cpp:449-489; D*T <= 64 only) or an external MILP solver.
This pipeline is the GPU-native counterpart the north star describes:
the MILP is assembled on the GPU (K1), its LP relaxation solved by PDHG (K3),
the relaxed diagonal R(d,t,t) seeds the randomised rounding of candidates
(K4, Philox keyed by (seed, global index)), and every batch is evaluated
exactly with the reference's semantics (K2: objective_value of the
completion, check_assignment families, integer budgets, decode legality).
The rounding incumbent is the first minimum over valid candidates in global
index order (solver.cpp:57-61), so shards on several GPUs reproduce one-GPU
results (shard.py).

Then a population of iterated local searches in R space (K4 xe_move_cubes:
recompute a parent where a consumer runs — with recomputation chains that
may cross devices —, drop a recomputation, move a computation; saves always
the canonical ones of the computations) starts from the best distinct
rounding candidates: every iteration evaluates `chain_n` neighbours of each
of the `chains` current schedules exactly (K2) and moves each chain to its
best valid neighbour when it improves, or after `stall` iterations without
improvement (a kick).  On config 2 (VGG-16, strict_free) this reaches the
reference's MILP optimum 128.32908933333337 (HiGHS via solve_external, 86 s)
bit for bit in ~2 s.

The LP objective is a lower bound on every schedule's objective
(binaries relaxed, same rows), reported beside the incumbent.  The whole
pipeline is one native call per GPU (xe_search, csrc/search.cu); this module
adds the multi-GPU exchange.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import LIB
from .api import ModelOptions, Problem, check

# a schedule is usable when check_assignment passes, every device stays
# within its integer budget (solver.cpp:237,249) and it decodes (schedule.cpp:40-129)
DEFAULT_MASK = _lib.F_CHECK_MASK | _lib.F_BUDGET | _lib.F_DECODE


@dataclass
class SearchResult:
    objective: float            # best valid objective (inf if none)
    index: int                  # global index of the best rounding candidate (-1 if none; the local
                                # search can still find a schedule from over-budget candidates)
    cube: Optional[np.ndarray]  # the final incumbent's canonical (R, S) cube, uint32 words
    peaks: Optional[np.ndarray]  # per-device peak bytes of the incumbent
    lp_bound: Optional[float]   # certified lower bound from the PDHG duals (Lagrangian value), None without LP
    lp_certified: bool
    n_evaluated: int
    n_valid: int                # valid rounding candidates
    ls_improvements: int = 0    # improvements of the incumbent found by the local search
    rounding_objective: float = float("inf")  # best rounding candidate alone
    time_limited: bool = False  # time_limit_ms cut the search short (on some rank)


def search(problem: Problem, opts: Optional[ModelOptions] = None, n_per_round: int = 1 << 18,
           rounds: int = 4, seed: int = 1, edits: int = 3, use_lp: bool = True,
           valid_mask: int = DEFAULT_MASK, first: int = 0, lp_tol: float = 1e-6,
           distributed: bool = False, chains: int = 256, chain_n: int = 1024, chain_iters: int = 200,
           max_moves: int = 4, stall: int = 15, canonical: bool = True,
           time_limit_ms: int = 0) -> SearchResult:
    """One native call (xe_search, csrc/search.cu) per GPU.
    distributed=True (torch.distributed initialised, one process per GPU):
    rank r rounds global index blocks (round * world + r) * n_per_round and
    runs its own local-search population (seeded by (seed, rank)); the
    rounding incumbent is the global first minimum (shard.exchange_best),
    the final schedule the best over ranks (lowest rank on ties), replacing
    the rounding incumbent only when strictly better, broadcast from the rank
    holding it.  canonical=True gives each rounded candidate the canonical
    saves of its computations; chains=0 skips the local search."""
    import ctypes as C
    import torch
    rank, world = 0, 1
    if distributed:
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
    opts = opts or ModelOptions()
    so = _lib.SearchOpts()
    _lib.LIB.xe_search_opts_default(C.byref(so))
    so.n_per_round, so.rounds, so.edits, so.seed = n_per_round, rounds, edits, seed
    so.use_lp, so.lp_tol, so.valid_mask, so.canonical = int(use_lp), lp_tol, valid_mask, int(canonical)
    so.chains, so.chain_n, so.chain_iters, so.max_moves, so.stall = chains, chain_n, chain_iters, max_moves, stall
    so.first, so.rank, so.world, so.time_limit_ms = first, rank, world, time_limit_ms
    res = _lib.SearchResult()
    cube = np.zeros(problem.cube_words, np.uint32)
    peaks = np.zeros(problem.D, np.int64)
    stream = torch.cuda.current_stream().cuda_stream
    check(_lib.LIB.xe_search(problem.handle, C.byref(opts.c()), C.byref(so), C.byref(res),
                             cube.ctypes.data, peaks.ctypes.data, C.c_void_p(stream)))
    obj, index, n_valid = res.objective, res.index, res.n_valid
    rounding, n_eval, impr = res.rounding_objective, res.n_evaluated, res.improvements
    if world > 1:
        import torch.distributed as dist
        from .shard import exchange_best, NONE
        inc = exchange_best(res.rounding_objective, res.index, res.n_valid, offset=0, device="cuda")
        win = exchange_best(res.objective, rank if math.isfinite(res.objective) else -1, 0, offset=0, device="cuda")
        owner = torch.tensor([rank if (res.index >= 0 and res.index == inc.index) else NONE],
                             dtype=torch.int64, device="cuda")
        dist.all_reduce(owner, op=dist.ReduceOp.MIN)
        tot = torch.tensor([res.n_evaluated, res.improvements], dtype=torch.int64, device="cuda")
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        n_eval, impr = int(tot[0].item()), int(tot[1].item())
        rounding, index, n_valid = inc.obj, inc.index, inc.n_valid
        if inc.index < 0 and win.index < 0:
            obj = float("inf")
        else:
            src = win.index if (inc.index < 0 or win.obj < inc.obj) else int(owner.item())
            obj = min(win.obj, inc.obj)
            buf = torch.from_numpy(np.concatenate([cube.view(np.int32), peaks.view(np.int32)])).cuda()
            dist.broadcast(buf, src=src)
            h = buf.cpu().numpy()
            cube = h[:problem.cube_words].copy().view(np.uint32)
            peaks = h[problem.cube_words:].copy().view(np.int64)
    has = math.isfinite(obj)
    limited = bool(res.time_limited)
    if world > 1:
        t = torch.tensor([int(limited)], dtype=torch.int64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        limited = bool(t.item())
    return SearchResult(obj, index, cube if has else None, peaks if has else None,
                        res.lp_bound if res.has_lp else None, bool(res.lp_certified), n_eval, n_valid, impr,
                        rounding, limited)


@dataclass
class PlacementSearchResult:
    objective: float             # best valid save-all (or minimal-save) objective, inf if none
    dev: Optional[np.ndarray]    # its device vector [T]
    peaks: Optional[np.ndarray]  # its per-device peaks
    random_objective: float      # best of the random sample alone
    n_evaluated: int
    improvements: int


def search_placements(problem: Problem, n_random: int = 1 << 22, chains: int = 256, chain_n: int = 1024,
                      iters: int = 100, max_moves: int = 4, stall: int = 15, seed: int = 1, policy: int = 0,
                      valid_mask: int = _lib.F_CHECK_MASK | _lib.F_BUDGET) -> PlacementSearchResult:
    """Best placement where the D^T sweep of assignment_oracle (solver.cpp:44-75,
    capped at 4e6 placements) cannot go — config 5 has 8^2000: K2b scores
    `n_random` uniform placements (xe_random_placements), the best distinct
    valid ones seed `chains` iterated local searches whose neighbours change
    the device of 1..max_moves random ops (to a device that can run them;
    K4 xe_move_placements);
    each iteration scores chains x chain_n neighbours exactly (K2b) and a
    chain moves to its best valid neighbour when it improves, or after
    `stall` iterations without improvement."""
    import ctypes as C
    import torch
    from .api import evaluate_placements, move_placements, random_placements
    dev = random_placements(problem, n_random, seed)
    r = evaluate_placements(problem, dev, policy=policy, valid_mask=valid_mask)
    score = torch.where((r.flags & valid_mask) == 0, r.obj, torch.full_like(r.obj, float("inf")))
    rand_best = float(score.min().item())
    if not np.isfinite(rand_best):
        return PlacementSearchResult(float("inf"), None, None, rand_best, n_random, 0)
    v, i = torch.sort(score)
    keep, last = [], None
    for val, idx in zip(v[:16 * chains].tolist(), i[:16 * chains].tolist()):
        if not np.isfinite(val):
            break
        if val != last:
            keep.append(idx)
            last = val
        if len(keep) == chains:
            break
    sel = torch.tensor([keep[k % len(keep)] for k in range(chains)], device="cuda")
    bases, cur = dev[sel].clone(), score[sel].clone()
    del dev, r, score
    P, M = chains, chain_n
    stalled = torch.zeros(P, dtype=torch.int32, device="cuda")
    k0 = int(torch.argmin(cur))
    best = cur[k0:k0 + 1].clone()            # device scalar: the incumbent
    best_dev = bases[k0].clone()
    improvements = torch.zeros(1, dtype=torch.int32, device="cuda")
    n_eval = n_random
    nb = torch.empty((P * M, problem.T), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for it in range(iters):
        move_placements(problem, bases, P * M, seed ^ 0x9E3779B9, first=it * P * M, max_moves=max_moves, out=nb)
        r = evaluate_placements(problem, nb, policy=policy, valid_mask=valid_mask, best=False)
        n_eval += P * M
        # chain control on the device (xe_placement_chains_step): no host sync per iteration
        check(LIB.xe_placement_chains_step(problem.handle, C.c_void_p(r.obj.data_ptr()),
                                           C.c_void_p(r.flags.data_ptr()), valid_mask, C.c_void_p(nb.data_ptr()),
                                           P, M, stall, C.c_void_p(bases.data_ptr()), C.c_void_p(cur.data_ptr()),
                                           C.c_void_p(stalled.data_ptr()), C.c_void_p(best.data_ptr()),
                                           C.c_void_p(best_dev.data_ptr()), C.c_void_p(improvements.data_ptr()),
                                           C.c_void_p(stream)))
        del r
    best = float(best.item())
    improvements = int(improvements.item())
    r1 = evaluate_placements(problem, best_dev.unsqueeze(0).contiguous(), policy=policy, valid_mask=valid_mask)
    assert r1.best_obj == best, (r1.best_obj, best)
    return PlacementSearchResult(best, best_dev.cpu().numpy(), r1.peak.cpu().numpy()[0], rand_best, n_eval,
                                 improvements)
