# SPDX-License-Identifier: Apache-2.0
"""K2a rate by candidate mix (VGG-16, 4 M candidates, CUDA events): how much
of the streaming evaluator's time the deferred timesteps take."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2212_09290_b200 as xe  # noqa: E402
from bench import configs  # noqa: E402

p = xe.Problem.from_json(configs.vgg16_doc())
n = 4_000_000
for edits, perturb in ((0, 0.0), (3, 0.0), (3, 0.1), (6, 0.1)):
    il = xe.cubes_to_il(p, xe.round_cubes(p, n, 2212, edits=edits, perturb=perturb))
    for _ in range(3):
        xe.evaluate_cubes_il(p, il, n, best=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        xe.evaluate_cubes_il(p, il, n, best=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"edits={edits} perturb={perturb}: {n / ms / 1e3:.1f} M cand/s", flush=True)
    del il
