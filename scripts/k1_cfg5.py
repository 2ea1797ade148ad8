# SPDX-License-Identifier: Apache-2.0
"""Config 5 (random 2000-op DAG, D = 8): K1 assembles the full MILP on one
B200 (1.18 G rows, 5.8 G nonzeros, ~120 GB of device CSR) — the reference
cannot build it in host RAM.  Checks the shape against the
closed-form family sizes and the CSR invariants, chunked
on the device."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_09290_b200 as xe  # noqa: E402
from bench import configs  # noqa: E402

p = xe.Problem.from_json(configs.random2000_doc())
T, D, E = p.T, p.D, p.E
FE = E + T
want = {"EQ8": 2 * T, "EQ9": 1, "EQ11": D * (T - 1) * T, "EQ12": D * T * E, "EQ13": D * T, "EQ14": D * T * (T - 1),
        "EQ16_LO": D * T * FE, "EQ16_HI": D * T * FE, "Z_LINK": 3 * D * T * T, "P_LINK": T * E * D * (D - 1)}
t0 = time.time()
m = xe.build_model(p)
torch.cuda.synchronize()
wall = time.time() - t0
print(f"cfg5 K1: rows {m.n_rows:,} cols {m.n_cols:,} nnz {m.nnz:,}  device {m.build_ms():.1f} ms  wall {wall:.1f} s  "
      f"memory {torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9:.1f} GB in use", flush=True)
assert (m.n_rows, m.n_cols, m.nnz) == (1181908001, 926336000, 5807616208), (m.n_rows, m.n_cols, m.nnz)
for k, v in want.items():
    assert m.tag_rows[k] == v, (k, m.tag_rows[k], v)
a = m.device_arrays()
rp, col, val = a["row_ptr"], a["col"], a["val"]
assert int(rp[0]) == 0 and int(rp[-1]) == m.nnz
step = 1 << 27
for lo in range(0, m.n_rows, step):
    hi = min(m.n_rows, lo + step)
    assert bool((rp[lo + 1:hi + 1] >= rp[lo:hi]).all()), lo
for lo in range(0, m.nnz, step):
    c = col[lo:lo + step]
    assert int(c.min()) >= 0 and int(c.max()) < m.n_cols, lo
    assert bool(torch.isfinite(val[lo:lo + step]).all()), lo
# EQ13 rows carry T + 2 terms: U(d,t,0), S(d,t,i) for all i, R(d,t,0)
off = sum(want[k] for k in ("EQ8", "EQ9", "EQ11", "EQ12"))
lens = (rp[off + 1:off + want["EQ13"] + 1] - rp[off:off + want["EQ13"]])
assert bool((lens == T + 2).all()), lens[:4]
print("cfg5 K1 invariants ok (family sizes, monotone row_ptr, columns in range, finite values, EQ13 lengths)")
