# SPDX-License-Identifier: Apache-2.0
"""LP-relaxation values of the reference model (HiGHS via scipy.optimize.linprog)
for the K3 parity tests -> tests/golden/lp_values.json.

The model is the oracle's CSR (pinned byte-for-byte to the reference's
write_mps, tests/test_oracle_cpu.py); binaries relaxed to [0,1], FX 0, U in
[0, budget], P in [0,1].  Third-party solver: HiGHS 1.12.0 inside SciPy 1.18.1.
Usage: python scripts/gen_lp_golden.py [--big] [--unet]
  --big adds ResNet-50 cfg 3 (~11 min IPM); --unet computes only U-Net cfg 4
  (IPM) and merges it into the existing file.
"""
import json
import os
import sys
import time

import numpy as np
import scipy
from scipy.optimize import linprog
from scipy.sparse import csr_matrix

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import xo  # noqa: E402
from bench import configs  # noqa: E402

G = os.path.join(ROOT, "tests", "golden")


def lp_value(a, strict=False, energy=False, method="highs"):
    O = xo.Oracle()
    m = O.build_model(a, strict, energy)
    A = csr_matrix((m.val, m.col, m.row_ptr), shape=(m.n_rows, m.n_cols))
    sense = m.sense.view("S1").astype(str)
    le = sense == "L"
    ge = sense == "G"
    eq = sense == "E"
    A_ub = __import__("scipy.sparse", fromlist=["vstack"]).vstack([A[le], -A[ge]]).tocsr()
    b_ub = np.concatenate([m.rhs[le], -m.rhs[ge]])
    T, D, E = a.T, a.D, a.E
    FE = E + T
    firstU = 3 * D * T * T + D * T * FE
    firstP = firstU + D * T * T
    ub = np.ones(m.n_cols)
    ub[m.fixed.astype(bool)] = 0.0
    for d in range(D):
        ub[firstU + d * T * T: firstU + (d + 1) * T * T] = a.budget[d]
    t0 = time.time()
    r = linprog(m.obj, A_ub=A_ub, b_ub=b_ub, A_eq=A[eq], b_eq=m.rhs[eq],
                bounds=np.stack([np.zeros(m.n_cols), ub], 1), method=method)
    assert r.status == 0, r.message
    return float(r.fun), time.time() - t0


def main():
    out = {"solver": f"HiGHS via scipy {scipy.__version__} linprog"}
    path = os.path.join(G, "lp_values.json")
    if os.path.exists(path):
        out.update(json.load(open(path)))
    cases = {
        "chain3": (xo.arrays_from_json(open(os.path.join(G, "problems", "chain3.json")).read()), False, False),
        "fig2": (xo.arrays_from_json(configs.fig2_doc()), False, False),
        "fig2_strict": (xo.arrays_from_json(configs.fig2_doc()), True, False),
        "fig2_energy": (xo.arrays_from_json(open(os.path.join(G, "problems", "fig2_energy.json")).read()), False, True),
        "vgg16": (xo.arrays_from_json(configs.vgg16_doc()), False, False),
    }
    lm = xo.arrays_from_json(open(os.path.join(G, "problems", "chain_lowmem.json")).read())
    full = int(lm.mass.sum())
    cases["chain_lowmem@25"] = (lm.with_budgets([full * 25 // 100]), False, False)
    for s in range(1, 6):
        cases[f"rand{s}"] = (xo.arrays_from_json(configs.random_small_doc(s)), False, False)
    if "--unet" in sys.argv:
        cases = {}
        a = xo.arrays_from_json(configs.unet_doc())
        v, dt = lp_value(a, method="highs-ipm")
        out["unet"] = {"lp": v, "seconds": dt, "method": "highs-ipm"}
        print("unet", v, dt, flush=True)
    for k, (a, strict, en) in cases.items():
        v, dt = lp_value(a, strict, en)
        out[k] = {"lp": v, "seconds": dt}
        print(k, v, f"{dt:.2f}s", flush=True)
    if "--big" in sys.argv:
        a = xo.arrays_from_json(configs.resnet50_doc())
        v, dt = lp_value(a, method="highs-ipm")
        out["resnet50"] = {"lp": v, "seconds": dt, "method": "highs-ipm"}
        print("resnet50", v, dt, flush=True)
    json.dump(out, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
