import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_2212_09290_b200 as xe
from bench import configs
from cubegen import unpack
p = xe.Problem.from_json(configs.vgg16_doc())
c = xe.round_cubes(p, 100000, 2212, edits=3, perturb=0.1).cpu().numpy().view(np.uint32)
R, S = unpack(c, p.D, p.T)   # [n, D, T, T]
n, D, T = R.shape[0], p.D, p.T
diag = np.arange(T)
onD = R[:, :, diag, diag]                   # [n, D, T]
cnt = onD.sum(axis=1)
off = R.sum(axis=(1, 3)) - cnt              # off-diagonal bits per t
nonfast = (off > 0) | (cnt != 1)
Z = R | S
eq11 = np.zeros((n, T), bool)
eq11[:, 1:] = ((S[:, :, 1:, :] & ~Z[:, :, :-1, :]).sum(axis=(1, 3)) > 0)
print("candidates", n, "non-fast timesteps per candidate", nonfast.sum(1).mean(), "eq11 timesteps", eq11.sum(1).mean())
print("frac candidates with any non-fast", (nonfast.sum(1) > 0).mean())
print("rows with >=2 computations per candidate", (R.sum(axis=3) >= 2).sum(axis=(1, 2)).mean())
print("hist non-fast", np.bincount(nonfast.sum(1))[:12])
