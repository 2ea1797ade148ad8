"""K4 generation rate (round_cubes, VGG-16 cfg 2 bench mix: 3 edits, 10 % flips)
and ResNet-50 (LP-free uniform placements, 3 edits): CUDA-event time per
launch, plus a digest of the cubes (unchanged across kernel revisions)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2212_09290_b200 as xe  # noqa: E402
from bench import configs  # noqa: E402

for name, n in (("vgg16", 1 << 21), ("resnet50", 1 << 17)):
    p = xe.Problem.from_json(configs.CONFIGS[name]())
    for _ in range(3):
        c = xe.round_cubes(p, n, 2212, edits=3, perturb=0.1)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c = xe.round_cubes(p, n, 2212, edits=3, perturb=0.1)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[2]
    dig = hashlib.sha256(c.cpu().numpy().tobytes()).hexdigest()[:16]
    print(f"{name} n={n} {ms:.2f} ms {n / ms / 1e3:.1f} M cand/s digest {dig}", flush=True)
