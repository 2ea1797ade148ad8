# SPDX-License-Identifier: Apache-2.0
"""Exercise the multi-rank search path (torchrun, any backend): every rank
must return the same schedule, re-scored to the same objective bits.
XE_DIST_BACKEND=gloo with 2 ranks on one GPU checks the code path only."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200.search import search  # noqa: E402
from bench import configs  # noqa: E402
from bench.dist import init_dist  # noqa: E402

local = init_dist(int(os.environ.get("LOCAL_RANK", "0")))
rank, world = dist.get_rank(), dist.get_world_size()
p = xe.Problem.from_json(configs.vgg16_doc(), device=local)
opts = xe.ModelOptions(strict_free=True)
r = search(p, opts, n_per_round=1 << 18, rounds=2, edits=6, seed=3, distributed=True, chain_iters=30)
re = xe.evaluate_cubes(p, torch.from_numpy(r.cube.view(np.int32)).cuda().unsqueeze(0), opts)
assert re.obj[0].item() == r.objective, (re.obj[0].item(), r.objective)
t = torch.tensor([r.objective, float(r.index), float(r.cube.astype(np.int64).sum())], dtype=torch.float64).cuda()
g = [torch.zeros_like(t) for _ in range(world)]
dist.all_gather(g, t)
assert all(torch.equal(g[0], x) for x in g), g
if rank == 0:
    print(f"world {world}: objective {r.objective!r} rounding {r.rounding_objective!r} index {r.index} "
          f"valid {r.n_valid} evaluated {r.n_evaluated} peaks {r.peaks.tolist()} - identical on all ranks")
dist.destroy_process_group()
