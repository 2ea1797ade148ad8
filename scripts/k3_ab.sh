# K3 A/B: lib (A) vs lib_alt (B) on the VGG-16 / ResNet-50 / U-Net LPs to 1e-7 (iterations, time)
python -m pytest tests/test_pdhg_gpu.py -x -q 2>&1 | tail -2
for L in lib lib_alt; do
  XE_LIB=paper_2212_09290_b200/$L/libxengine_b200.so python - <<'PY'
import os, time, paper_2212_09290_b200 as xe
from bench import configs
for name in ("fig2", "vgg16", "resnet50", "unet"):
    m = xe.build_model(xe.Problem.from_json(configs.CONFIGS[name]() if name != "fig2" else configs.fig2_doc()))
    t = time.time(); r = xe.pdhg_solve(m, tol=1e-7, max_iters=1000000)
    print(os.environ["XE_LIB"].split("/")[1], name, r.iters, r.restarts, r.converged, r.certified, repr(r.primal_obj),
          f"{time.time()-t:.2f}s", f"solve {r.solve_ms/1e3:.2f}s", f"{r.ms_per_iter*1e3:.1f} us/it", flush=True)
PY
done
