python -m pytest tests/test_pdhg_gpu.py -x -q 2>&1 | tail -3
for L in lib lib_alt; do
  echo "== $L"
  XE_LIB=paper_2212_09290_b200/$L/libxengine_b200.so python scripts/prof_k1k3.py k3 4096
  XE_LIB=paper_2212_09290_b200/$L/libxengine_b200.so python scripts/prof_k1k3.py k3r 4096
done
python - <<'PY'
import time, paper_2212_09290_b200 as xe
from bench import configs
m = xe.build_model(xe.Problem.from_json(configs.resnet50_doc()))
t = time.time(); r = xe.pdhg_solve(m, tol=1e-7, max_iters=1000000)
print("resnet full", r.iters, r.converged, r.certified, r.primal_obj, f"{time.time()-t:.2f}s", f"{r.ms_per_iter*1e3:.1f} us/it")
PY
