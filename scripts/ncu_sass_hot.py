# SPDX-License-Identifier: Apache-2.0
"""Hot SASS of a kernel: per-instruction executed counts (ncu source page,
--print-source sass) with the disassembly, for reading the steady-state loop.
usage: python scripts/ncu_sass_hot.py REPORT.ncu-rep [min_share_percent]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.02
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ai, si, ie = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
te = h.index("Thread Instructions Executed") if "Thread Instructions Executed" in h else None
data = []
for r in rows[2:]:
    try:
        v = float(r[ie] or 0)
    except ValueError:
        continue
    th = float(r[te] or 0) if te is not None else 0.0
    data.append((r[ai], r[si], v, th))
tot = sum(d[2] for d in data)
print(f"total warp-instructions {tot:.4g}")
for a, src, v, th in data:
    if v / tot * 100 >= thr:
        print(f"{a} {v / tot * 100:6.3f}% lanes={th / v if v else 0:5.1f}  {src}")
