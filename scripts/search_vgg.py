# SPDX-License-Identifier: Apache-2.0
"""Config 2 (VGG-16, strict_free): how close the LP-guided search + local
search gets to the reference's MILP optimum 128.32908933333337 ms (HiGHS via
solve_external)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200.search import search  # noqa: E402
from bench import configs  # noqa: E402

p = xe.Problem.from_json(configs.vgg16_doc())
for edits, ls in ((6, 0), (8, 0), (12, 0), (6, 100), (8, 200)):
    t0 = time.time()
    r = search(p, xe.ModelOptions(strict_free=True), n_per_round=1 << 20, rounds=8, edits=edits, seed=edits,
               ls_rounds=ls, ls_n=1 << 16, ls_edits=2)
    print(f"edits={edits} ls_rounds={ls}: best {r.objective!r} (LP {r.lp_bound:.6f}, MILP 128.32908933333337) "
          f"valid {r.n_valid}/{r.n_evaluated} ls+{r.ls_improvements} peaks {[int(x) for x in r.peaks]} "
          f"{time.time() - t0:.1f}s", flush=True)
