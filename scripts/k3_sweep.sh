# K3 timing on the VGG-16 and ResNet-50 LPs (4096 iterations each) and the full ResNet-50 solve
python scripts/prof_k1k3.py k3 4096 | tail -1
python scripts/prof_k1k3.py k3r 4096 | tail -1
python - <<'PY'
import time, paper_2212_09290_b200 as xe
from bench import configs
m = xe.build_model(xe.Problem.from_json(configs.resnet50_doc()))
t = time.time(); r = xe.pdhg_solve(m, tol=1e-7, max_iters=1000000)
print("resnet full", r.iters, r.converged, r.certified, r.primal_obj, f"{time.time()-t:.2f}s", f"{r.ms_per_iter*1e3:.1f} us/it")
PY
