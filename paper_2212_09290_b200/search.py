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
The incumbent is the first minimum over valid candidates in global index
order (solver.cpp:57-61), so shards on several GPUs reproduce one-GPU
results (shard.py).

The LP objective is a lower bound on every schedule's objective
(binaries relaxed, same rows), reported beside the incumbent.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .api import ModelOptions, Problem, build_model, evaluate_cubes, mutate_cubes, pdhg_solve, round_cubes

# a schedule is usable when check_assignment passes, every device stays
# within its integer budget (solver.cpp:237,249) and it decodes (schedule.cpp:40-129)
DEFAULT_MASK = _lib.F_CHECK_MASK | _lib.F_BUDGET | _lib.F_DECODE


@dataclass
class SearchResult:
    objective: float            # best valid objective (inf if none)
    index: int                  # global candidate index of the incumbent (-1 if none)
    cube: Optional[np.ndarray]  # the incumbent's canonical (R, S) cube, uint32 words
    peaks: Optional[np.ndarray]  # per-device peak bytes of the incumbent
    lp_bound: Optional[float]   # PDHG LP relaxation value (lower bound), None without LP
    lp_certified: bool
    n_evaluated: int
    n_valid: int
    ls_improvements: int = 0    # incumbent improvements found by the local search


def search(problem: Problem, opts: Optional[ModelOptions] = None, n_per_round: int = 1 << 18,
           rounds: int = 4, seed: int = 1, edits: int = 3, use_lp: bool = True,
           valid_mask: int = DEFAULT_MASK, first: int = 0, lp_tol: float = 1e-6,
           distributed: bool = False, ls_rounds: int = 0, ls_n: int = 1 << 16,
           ls_edits: int = 2) -> SearchResult:
    """distributed=True (torch.distributed initialised, one process per GPU):
    rank r evaluates global index blocks (round * world + r) * n_per_round,
    the incumbent is exchanged with shard.exchange_best; every rank returns
    the global result (the LP is solved on every rank: PDHG is deterministic)."""
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
    best_obj, best_idx, n_valid = float("inf"), -1, 0
    for r in range(rounds):
        lo = first + (r * world + rank) * n_per_round
        cubes = round_cubes(problem, n_per_round, seed, first=lo, edits=edits, perturb=0.0, x=x_dev)
        res = evaluate_cubes(problem, cubes, opts, valid_mask=valid_mask, outputs=False)
        n_valid += res.n_valid
        if res.best_index >= 0 and res.best_obj < best_obj:  # rounds ascend in index: strict <
            best_obj, best_idx = res.best_obj, lo + res.best_index
        del cubes
    if world > 1:
        from .shard import exchange_best
        inc = exchange_best(best_obj, best_idx, n_valid, offset=0, device="cuda")
        best_obj, best_idx, n_valid = inc.obj, inc.index, inc.n_valid
    cube = peaks = None
    n_eval = rounds * n_per_round * world
    improvements = 0
    if best_idx >= 0:
        c = round_cubes(problem, 1, seed, first=best_idx, edits=edits, perturb=0.0, x=x_dev)
        r1 = evaluate_cubes(problem, c, opts, valid_mask=valid_mask)
        assert r1.best_obj == best_obj, (r1.best_obj, best_obj)
        # K4 local search: hill-climb over neighbours of the incumbent (one
        # op moved with its saves, drop-and-recompute edits), K2 scoring
        inc = c[0].clone()
        for it in range(ls_rounds):
            nb = mutate_cubes(problem, inc, ls_n, seed ^ 0x5EED, first=it * ls_n, edits=ls_edits)
            r2 = evaluate_cubes(problem, nb, opts, valid_mask=valid_mask, outputs=False)
            n_eval += ls_n
            if r2.best_index >= 0 and r2.best_obj < best_obj:
                best_obj, inc = r2.best_obj, nb[r2.best_index].clone()
                improvements += 1
            del nb
        r1 = evaluate_cubes(problem, inc.unsqueeze(0), opts, valid_mask=valid_mask)
        assert r1.best_obj == best_obj, (r1.best_obj, best_obj)
        cube = inc.cpu().numpy().view(np.uint32)
        peaks = r1.peak.cpu().numpy()[0]
    return SearchResult(best_obj, best_idx, cube, peaks, lp_val, cert, n_eval, n_valid, improvements)
