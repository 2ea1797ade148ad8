"""LP-guided K4 rounding (x from the PDHG relaxation): digest of the cubes and
the rate, for comparing library builds (cubes must be identical)."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2212_09290_b200 as xe  # noqa: E402
from bench import configs  # noqa: E402

for name, n in (("vgg16", 1 << 20), ("resnet50", 1 << 17)):
    p = xe.Problem.from_json(configs.CONFIGS[name]())
    m = xe.build_model(p)
    lp = xe.pdhg_solve(m, tol=1e-4, max_iters=20000, return_x=True)
    x = torch.from_numpy(lp.x).cuda()
    out = torch.empty((n, p.cube_words), dtype=torch.int32, device="cuda")
    for _ in range(2):
        xe.round_cubes(p, n, 2212, edits=3, perturb=0.0, x=x, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        xe.round_cubes(p, n, 2212, edits=3, perturb=0.0, x=x, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[2]
    print(f"{name} LP-guided n={n} {ms:.2f} ms {n / ms / 1e3:.1f} M cand/s digest "
          f"{hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]}", flush=True)
