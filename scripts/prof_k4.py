# SPDX-License-Identifier: Apache-2.0
"""Profiling driver for ncu: the K4 kernels of one search (VGG-16 cfg 2,
strict_free): rounding, canonical saves / R-space moves, chain selection."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200.search import search  # noqa: E402
from bench import configs  # noqa: E402

p = xe.Problem.from_json(configs.vgg16_doc())
r = search(p, xe.ModelOptions(strict_free=True), n_per_round=1 << 20, rounds=1, edits=6, seed=1, chain_iters=4)
print("k4 search", r.objective, r.n_evaluated)
