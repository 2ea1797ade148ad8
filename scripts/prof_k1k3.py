# SPDX-License-Identifier: Apache-2.0
"""Profiling driver for ncu: K1 assembly of the ResNet-50 cfg 3 model and a
fixed number of PDHG iterations on the VGG-16 cfg 2 LP (the kernels of the
bench's k1_build / pdhg objects)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_09290_b200 as xe  # noqa: E402
from bench import configs  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
if which in ("k1", "both"):
    m = xe.build_model(xe.Problem.from_json(configs.resnet50_doc()))
    print("k1 resnet50", m.n_rows, m.n_cols, m.nnz, f"{m.build_ms():.2f} ms")
if which in ("k3", "both"):
    m = xe.build_model(xe.Problem.from_json(configs.vgg16_doc()))
    r = xe.pdhg_solve(m, tol=1e-12, max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 2048)
    print("k3 vgg16", r.iters, f"{r.ms_per_iter * 1e3:.2f} us/iter", r.primal_obj)
if which == "k3r":
    m = xe.build_model(xe.Problem.from_json(configs.resnet50_doc()))
    print("model", m.n_rows, m.n_cols, m.nnz)
    r = xe.pdhg_solve(m, tol=1e-12, max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 2048)
    print("k3 resnet50", r.iters, f"{r.ms_per_iter * 1e3:.2f} us/iter", r.primal_obj)
