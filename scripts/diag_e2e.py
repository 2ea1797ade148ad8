# SPDX-License-Identifier: Apache-2.0
"""Diagnose the end-to-end (host buffer) path: H2D bandwidth from pinned
memory via torch vs. through the C ABI."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2212_09290_b200 as xe
from bench import configs
prob = xe.Problem.from_json(configs.vgg16_doc())
n = 2_000_000
dev = xe.round_cubes(prob, n, seed=1)
host = torch.empty_like(dev, device="cpu").pin_memory()
host.copy_(dev); torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter(); d2 = host.to("cuda", non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"torch pinned H2D {host.numel()*4/(t1-t0)/1e9:.1f} GB/s")
hnp = host.numpy()
for _ in range(3):
    t0 = time.perf_counter(); r = xe.evaluate_cubes_host(prob, hnp, outputs=False); t1 = time.perf_counter()
    print(f"xe_eval_cubes_host pinned: {t1-t0:.3f}s  {n/(t1-t0)/1e6:.1f} Mcand/s  {host.numel()*4/(t1-t0)/1e9:.1f} GB/s")
pg = np.array(hnp)
t0 = time.perf_counter(); r = xe.evaluate_cubes_host(prob, pg, outputs=False); t1 = time.perf_counter()
print(f"xe_eval_cubes_host pageable: {t1-t0:.3f}s")
t0 = time.perf_counter(); r2 = xe.evaluate_cubes(prob, dev); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"device eval: {t1-t0:.3f}s best {r2.best_index} vs host {r.best_index}")
