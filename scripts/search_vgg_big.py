# SPDX-License-Identifier: Apache-2.0
"""Config 2 (VGG-16, strict_free): a larger LP-guided search + local search
against the reference's MILP optimum 128.32908933333337 ms."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200.search import search  # noqa: E402
from bench import configs  # noqa: E402

p = xe.Problem.from_json(configs.vgg16_doc())
best = None
for edits in (5, 6, 7, 9):
    t0 = time.time()
    r = search(p, xe.ModelOptions(strict_free=True), n_per_round=1 << 22, rounds=16, edits=edits, seed=100 + edits,
               ls_rounds=300, ls_n=1 << 18, ls_edits=3)
    print(f"edits={edits}: best {r.objective!r} valid {r.n_valid} evaluated {r.n_evaluated} ls+{r.ls_improvements} "
          f"peaks {[int(x) for x in r.peaks]} {time.time() - t0:.1f}s", flush=True)
