# SPDX-License-Identifier: Apache-2.0
"""One small invocation of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck):  K1 build + CSC, K3 PDHG (a few hundred
iterations), K4 rounding + moves + placements, K2a streaming + reference-order
evaluators (fig2, VGG-16, ResNet-50 shapes), K2b placements (both kernels) + oracle,
the search, solve_exact, schedule decode / validate / replay, device MPS."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2212_09290_b200 as xe  # noqa: E402
from paper_2212_09290_b200 import schedule as sch  # noqa: E402
from paper_2212_09290_b200.search import search  # noqa: E402
from bench import configs  # noqa: E402

fig2 = open(os.path.join(ROOT, "tests", "golden", "problems", "fig2.json")).read()
for name, doc, n in (("fig2", fig2, 300), ("vgg16", configs.vgg16_doc(), 2048), ("resnet50", configs.resnet50_doc(), 256)):
    p = xe.Problem.from_json(doc)
    m = xe.build_model(p)
    m.write_mps()                                         # device MPS emission
    xe.build_model(p, xe.ModelOptions(quadratic_objective=True)).write_mps()  # QUADOBJ
    m.csc()
    lp = xe.pdhg_solve(m, tol=1e-3, max_iters=256, return_x=True)
    xe.round_cubes(p, min(n, 512), 9, edits=3, perturb=0.1, x=torch.from_numpy(lp.x).cuda())  # LP-guided K4
    cubes = xe.round_cubes(p, n, 7, edits=3, perturb=0.1)
    nb = xe.move_cubes(p, cubes[:4], 64, 3, max_moves=3)
    r = xe.evaluate_cubes(p, cubes)                       # streaming (fast) path + refine
    il = xe.cubes_to_il(p, cubes)
    xe.evaluate_cubes_il(p, il, n)
    p.set_exact_objective(True)
    xe.evaluate_cubes(p, nb)                              # reference-order kernels
    p.set_exact_objective(False)
    dev = xe.random_placements(p, 256, 5)
    xe.evaluate_placements(p, dev, policy=0)
    xe.evaluate_placements(p, dev, policy=1)
    s = sch.decode(p, cubes[:8].cpu().numpy().view(np.uint32))
    ok = [x for x in s if x.error is None]
    if ok:
        rep = sch.validate(p, ok)
        good = [x for x, v in zip(ok, rep) if not v]
        if good:
            sch.replay(p, good)
    print(name, "ok", r.best_obj, flush=True)
p5 = xe.Problem.from_json(configs.random2000_doc())
xe.evaluate_placements(p5, xe.random_placements(p5, 96, 3), policy=0)  # bit-sliced K2b (D = 8)
print("random2000 ok", flush=True)
p = xe.Problem.from_json(fig2)
xe.assignment_oracle(p)
print("exact", xe.solve_exact(p).objective)
print("search", search(p, n_per_round=1 << 10, rounds=1, chains=8, chain_n=32, chain_iters=2).objective)
torch.cuda.synchronize()
print("done")
