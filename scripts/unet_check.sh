python -m pytest tests/test_model_gpu.py -x -q -k mps_sha 2>&1 | tail -2
python - <<'PY'
import time, paper_2212_09290_b200 as xe
from bench import configs
m = xe.build_model(xe.Problem.from_json(configs.unet_doc()))
print("unet model", m.n_rows, m.n_cols, m.nnz, f"{m.build_ms():.2f} ms")
t = time.time(); r = xe.pdhg_solve(m, tol=1e-7, max_iters=1000000)
print("unet lp", r.iters, r.converged, r.certified, repr(r.primal_obj), r.dual_obj, f"{time.time()-t:.2f}s", f"{r.ms_per_iter*1e3:.1f} us/it")
PY
