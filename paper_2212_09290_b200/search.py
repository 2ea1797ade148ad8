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
(binaries relaxed, same rows), reported beside the incumbent.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .api import ModelOptions, Problem, build_model, evaluate_cubes, move_cubes, pdhg_solve, round_cubes

# a schedule is usable when check_assignment passes, every device stays
# within its integer budget (solver.cpp:237,249) and it decodes (schedule.cpp:40-129)
DEFAULT_MASK = _lib.F_CHECK_MASK | _lib.F_BUDGET | _lib.F_DECODE


@dataclass
class SearchResult:
    objective: float            # best valid objective (inf if none)
    index: int                  # global index of the best rounding candidate (-1 if none)
    cube: Optional[np.ndarray]  # the final incumbent's canonical (R, S) cube, uint32 words
    peaks: Optional[np.ndarray]  # per-device peak bytes of the incumbent
    lp_bound: Optional[float]   # PDHG LP relaxation value (lower bound), None without LP
    lp_certified: bool
    n_evaluated: int
    n_valid: int                # valid rounding candidates
    ls_improvements: int = 0    # improvements of the incumbent found by the local search
    rounding_objective: float = float("inf")  # best rounding candidate alone


def _valid_obj(res, valid_mask):
    import torch
    ok = (res.flags & valid_mask) == 0
    return torch.where(ok, res.obj, torch.full_like(res.obj, float("inf")))


def _merge_pool(pool_obj, pool_cubes, obj, cubes, k):
    """Best k distinct objective values of the pool plus a new batch."""
    import torch
    take = min(obj.numel(), 4 * k)
    v, i = torch.topk(obj, take, largest=False)
    cand_obj = torch.cat([pool_obj, v]) if pool_obj is not None else v
    cand_cubes = torch.cat([pool_cubes, cubes[i]]) if pool_cubes is not None else cubes[i]
    order = torch.argsort(cand_obj, stable=True)
    vals = cand_obj[order].tolist()
    keep, last = [], None
    for j, x in zip(order.tolist(), vals):
        if not np.isfinite(x):
            break
        if x != last:
            keep.append(j)
            last = x
        if len(keep) == k:
            break
    if not keep:
        return pool_obj, pool_cubes
    sel = torch.tensor(keep, device=cand_obj.device)
    return cand_obj[sel].clone(), cand_cubes[sel].clone()


def local_search(problem: Problem, opts: ModelOptions, bases, objs, iters: int = 100, chain_n: int = 1024,
                 seed: int = 1, max_moves: int = 4, stall: int = 15, valid_mask: int = DEFAULT_MASK):
    """Population of iterated local searches in R space from `bases`
    ([chains, cube_words] int32 CUDA, canonical saves) with objectives `objs`.
    Returns (best objective, best cube, improvements, evaluations)."""
    import torch
    P = bases.shape[0]
    dev = bases.device
    cur = objs.clone()
    best = float(cur.min().item())
    best_cube = bases[int(torch.argmin(cur))].clone()
    stalled = torch.zeros(P, dtype=torch.int32, device=dev)
    rows = torch.arange(P, device=dev) * chain_n
    improvements = 0
    for it in range(iters):
        nb = move_cubes(problem, bases, P * chain_n, seed, first=it * P * chain_n, max_moves=max_moves)
        r = evaluate_cubes(problem, nb, opts, valid_mask=valid_mask)
        v, j = _valid_obj(r, valid_mask).view(P, chain_n).min(1)
        better = v < cur
        take = better | ((stalled >= stall) & torch.isfinite(v))
        bases = torch.where(take[:, None], nb[rows + j], bases)
        cur = torch.where(take, v, cur)
        stalled = torch.where(take, torch.zeros_like(stalled), stalled + 1)
        b = float(cur.min().item())
        if b < best:
            best, best_cube = b, bases[int(torch.argmin(cur))].clone()
            improvements += 1
        del nb, r
    return best, best_cube, improvements, iters * P * chain_n


def search(problem: Problem, opts: Optional[ModelOptions] = None, n_per_round: int = 1 << 18,
           rounds: int = 4, seed: int = 1, edits: int = 3, use_lp: bool = True,
           valid_mask: int = DEFAULT_MASK, first: int = 0, lp_tol: float = 1e-6,
           distributed: bool = False, chains: int = 256, chain_n: int = 1024, chain_iters: int = 100,
           max_moves: int = 4, stall: int = 15, canonical: bool = True) -> SearchResult:
    """distributed=True (torch.distributed initialised, one process per GPU):
    rank r evaluates global index blocks (round * world + r) * n_per_round,
    the rounding incumbent is exchanged with shard.exchange_best, every rank
    runs its own local-search population (seeded by rank) and the best final
    schedule is broadcast from the lowest rank holding it; every rank returns
    the global result (the LP is solved on every rank: PDHG is deterministic).
    canonical=True replaces each rounded candidate's saves by the canonical
    saves of its computations (xe_move_cubes with no move) before evaluation.
    chains=0 skips the local search (T <= 256 for it)."""
    import torch
    rank, world = 0, 1
    if distributed:
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
    opts = opts or ModelOptions()
    x_dev, lp_val, cert = None, None, True
    if use_lp:
        model = build_model(problem, opts)
        lp = pdhg_solve(model, tol=lp_tol, max_iters=400000, return_x=True)
        x_dev = torch.from_numpy(lp.x).cuda()
        lp_val, cert = lp.primal_obj, lp.certified
    canonical = canonical and problem.T <= 256
    chains = chains if problem.T <= 256 else 0

    def candidates(lo, n):
        c = round_cubes(problem, n, seed, first=lo, edits=edits, perturb=0.0, x=x_dev)
        return move_cubes(problem, c, n, 0, max_moves=0, out=c) if canonical else c

    best_obj, best_idx, n_valid = float("inf"), -1, 0
    pool_obj = pool_cubes = None
    for r in range(rounds):
        lo = first + (r * world + rank) * n_per_round
        cubes = candidates(lo, n_per_round)
        res = evaluate_cubes(problem, cubes, opts, valid_mask=valid_mask, outputs=chains > 0)
        n_valid += res.n_valid
        if res.best_index >= 0 and res.best_obj < best_obj:  # rounds ascend in index: strict <
            best_obj, best_idx = res.best_obj, lo + res.best_index
        if chains > 0 and res.n_valid > 0:
            pool_obj, pool_cubes = _merge_pool(pool_obj, pool_cubes, _valid_obj(res, valid_mask), cubes, chains)
        del cubes, res
    if world > 1:
        from .shard import exchange_best
        inc = exchange_best(best_obj, best_idx, n_valid, offset=0, device="cuda")
        best_obj, best_idx, n_valid = inc.obj, inc.index, inc.n_valid
    n_eval = rounds * n_per_round * world
    rounding_obj = best_obj
    cube = peaks = None
    improvements = 0
    if best_idx >= 0:
        inc_cube = candidates(best_idx, 1)[0].clone()
        r1 = evaluate_cubes(problem, inc_cube.unsqueeze(0), opts, valid_mask=valid_mask)
        assert r1.best_obj == best_obj, (r1.best_obj, best_obj)
        if pool_obj is not None:
            P = pool_obj.numel()
            reps = (chains + P - 1) // P
            bases = pool_cubes.repeat(reps, 1)[:chains].contiguous()
            objs = pool_obj.repeat(reps)[:chains].contiguous()
            ls_obj, ls_cube, improvements, ev = local_search(
                problem, opts, bases, objs, iters=chain_iters, chain_n=chain_n,
                seed=(seed * 1000003 + rank) & 0xFFFFFFFFFFFF, max_moves=max_moves, stall=stall,
                valid_mask=valid_mask)
            n_eval += ev * world
            if ls_obj < best_obj:
                best_obj, inc_cube = ls_obj, ls_cube
        if world > 1:
            import torch.distributed as dist
            from .shard import exchange_best
            win = exchange_best(best_obj, rank, 0, offset=0, device="cuda")
            buf = inc_cube.contiguous().clone()
            dist.broadcast(buf, src=win.index)
            best_obj, inc_cube = win.obj, buf
        r1 = evaluate_cubes(problem, inc_cube.unsqueeze(0), opts, valid_mask=valid_mask)
        assert r1.best_obj == best_obj, (r1.best_obj, best_obj)
        cube = inc_cube.cpu().numpy().view(np.uint32)
        peaks = r1.peak.cpu().numpy()[0]
    return SearchResult(best_obj, best_idx, cube, peaks, lp_val, cert, n_eval, n_valid, improvements, rounding_obj)
