# SPDX-License-Identifier: Apache-2.0
"""Profiling driver for ncu (round 2): one workload per argument.
  eval_vgg    K2a streaming evaluator, VGG-16 cfg 2, 2 M K4 candidates (bench shape)
  eval_resnet K2a streaming evaluator, ResNet-50 cfg 3 (T=145, NW=3), 256 k rounded candidates
  place       K2b save-all placements, random2000 cfg 5, 1 M placements
  round       K4 round_cubes, VGG-16, 1 M candidates
  exact       solve_exact on fig2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2212_09290_b200 as xe  # noqa: E402
from bench import configs  # noqa: E402

which = sys.argv[1]
if which == "eval_vgg":
    p = xe.Problem.from_json(configs.vgg16_doc())
    n = 2_000_000
    il = xe.cubes_to_il(p, xe.round_cubes(p, n, 2212, edits=3, perturb=0.1))
    for _ in range(4):
        xe.evaluate_cubes_il(p, il, n, best=False)
elif which == "eval_resnet":
    p = xe.Problem.from_json(configs.resnet50_doc())
    n = 1 << 18
    il = xe.cubes_to_il(p, xe.round_cubes(p, n, 2212, edits=3, perturb=0.0))
    for _ in range(4):
        xe.evaluate_cubes_il(p, il, n, best=False)
elif which == "place":
    p = xe.Problem.from_json(configs.random2000_doc())
    dev = xe.random_placements(p, 1 << 20, 2212)
    for _ in range(4):
        xe.evaluate_placements(p, dev, policy=0)
elif which == "round":
    p = xe.Problem.from_json(configs.vgg16_doc())
    for _ in range(4):
        xe.round_cubes(p, 1 << 20, 2212, edits=3, perturb=0.1)
elif which == "exact":
    p = xe.Problem.from_json(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "problems",
                                               "fig2.json")).read())
    print(xe.solve_exact(p))
torch.cuda.synchronize()
print("done", which)
