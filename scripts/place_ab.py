"""K2b A/B: the bit-sliced save-all kernel against the warp-per-placement
kernel (XE_PLACE_SLICED=0) on config 5 (random2000, D=8): CUDA-event time
per launch and identical outputs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2212_09290_b200 as xe  # noqa: E402
from bench import configs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
p = xe.Problem.from_json(configs.random2000_doc())
dev = xe.random_placements(p, n, 2212)
res = {}
for mode in ("1", "0"):
    os.environ["XE_PLACE_SLICED"] = mode
    out = (torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty((n, p.D), dtype=torch.int64, device="cuda"),
           torch.empty(n, dtype=torch.int32, device="cuda"))
    r = xe.evaluate_placements(p, dev, policy=0, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        r = xe.evaluate_placements(p, dev, policy=0, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res[mode] = [t.clone() for t in out] + [r]
    print(f"sliced={mode} {ms:.2f} ms  {n / ms / 1e3:.1f} M placements/s  best={(r.best_obj, r.best_index, r.n_valid)}", flush=True)
a, b = res["1"], res["0"]
print("obj equal", torch.equal(a[0].view(torch.int64), b[0].view(torch.int64)), "peaks equal", torch.equal(a[1], b[1]),
      "flags equal", torch.equal(a[2], b[2]))
