# K3 A/B: coded SELL entries (default) vs scaled fp64 values (XE_PDHG_CODED=0)
# on the VGG-16 / ResNet-50 / U-Net LPs to 1e-7 (iterations, time), then the tests
for C in 1 0; do
  XE_PDHG_CODED=$C python - <<'PY'
import os, time, paper_2212_09290_b200 as xe
from bench import configs
for name in ("vgg16", "resnet50", "unet"):
    m = xe.build_model(xe.Problem.from_json(configs.CONFIGS[name]()))
    t = time.time(); r = xe.pdhg_solve(m, tol=1e-7, max_iters=1000000)
    print("coded=" + os.environ["XE_PDHG_CODED"], name, r.iters, r.restarts, r.converged, r.certified, repr(r.primal_obj),
          f"{time.time()-t:.2f}s", f"solve {r.solve_ms/1e3:.2f}s", f"{r.ms_per_iter*1e3:.2f} us/it", flush=True)
PY
done
python -m pytest tests/test_pdhg_gpu.py -x -q 2>&1 | tail -2
