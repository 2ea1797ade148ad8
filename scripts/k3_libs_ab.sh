#!/bin/bash
# K3 A/B over library builds: VGG-16 / ResNet-50 / U-Net LPs to 1e-7 (iterations, us per iteration)
for rep in 1 2; do
for lib in "$@"; do
  XE_LIB_LENIENT=1 XE_LIB=$PWD/$lib python - <<'PY'
import os, paper_2212_09290_b200 as xe
from bench import configs
for name in ("vgg16", "resnet50", "unet"):
    m = xe.build_model(xe.Problem.from_json(configs.CONFIGS[name]()))
    r = xe.pdhg_solve(m, tol=1e-7, max_iters=1000000)
    print(os.path.basename(os.environ["XE_LIB"]), name, r.iters, r.converged, r.certified, repr(r.primal_obj),
          f"{r.ms_per_iter*1e3:.2f} us/it", flush=True)
PY
done
done
