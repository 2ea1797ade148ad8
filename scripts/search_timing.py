import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2212_09290_b200 as xe
from bench import configs
from paper_2212_09290_b200.search import search
p = xe.Problem.from_json(configs.vgg16_doc())
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sr = search(p, xe.ModelOptions(strict_free=True), n_per_round=1 << 20, rounds=2, edits=6, seed=1)
    torch.cuda.synchronize(); print(os.environ.get("XE_ROUND_BATCH", "default"), sr.objective, time.perf_counter() - t0, flush=True)
pr = xe.Problem.from_json(configs.resnet50_doc())
torch.cuda.synchronize(); t0 = time.perf_counter(); c = xe.round_cubes(pr, 1 << 18, 1, edits=3); torch.cuda.synchronize()
print("resnet round 256k", (1 << 18) / (time.perf_counter() - t0) / 1e6, "M/s")
