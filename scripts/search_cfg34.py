# SPDX-License-Identifier: Apache-2.0
"""Configs 3-4 (ResNet-50 / U-Net training DAGs): the search's best schedule
against the PDHG LP lower bound, rounding alone vs with the R-space
local-search population."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200.search import search  # noqa: E402
from bench import configs  # noqa: E402

for name in sys.argv[1:] or ["resnet50", "unet"]:
    p = xe.Problem.from_json(configs.CONFIGS[name]())
    for chains, iters in ((0, 0), (256, 100), (256, 400)):
        t0 = time.time()
        r = search(p, n_per_round=1 << 16, rounds=4, edits=6, seed=1, chains=chains, chain_iters=iters,
                   chain_n=256)
        print(f"{name} chains={chains} iters={iters}: best {r.objective!r} rounding {r.rounding_objective!r} "
              f"LP {r.lp_bound:.5f} gap-to-LP {100 * (r.objective / r.lp_bound - 1):.2f}% evaluated {r.n_evaluated} "
              f"ls+{r.ls_improvements} peaks {[int(x) for x in r.peaks]} {time.time() - t0:.1f}s", flush=True)
