# SPDX-License-Identifier: Apache-2.0
"""Config 2 (VGG-16, strict_free): the search (K1 -> K3 -> K4 rounding ->
R-space local-search population, K2 scoring) against the reference's MILP
optimum 128.32908933333337 ms (HiGHS via solve_external), over
several seeds; rounding-only runs (chains=0) for comparison."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200.search import search  # noqa: E402
from bench import configs  # noqa: E402

OPT = 128.32908933333337
p = xe.Problem.from_json(configs.vgg16_doc())
opts = xe.ModelOptions(strict_free=True)
search(p, opts, n_per_round=1 << 16, rounds=1, chain_iters=2)  # warm-up (module load, graphs)
for seed in range(1, 9):
    for chains in (0, 256):
        t0 = time.time()
        r = search(p, opts, n_per_round=1 << 20, rounds=2, edits=6, seed=seed, chains=chains)
        dt = time.time() - t0
        print(f"seed={seed} chains={chains}: best {r.objective!r} (gap {100 * (r.objective / OPT - 1):.4f}%, "
              f"rounding {r.rounding_objective!r}, LP {r.lp_bound:.6f}) evaluated {r.n_evaluated} "
              f"ls+{r.ls_improvements} peaks {[int(x) for x in r.peaks]} {dt:.1f}s", flush=True)
