# SPDX-License-Identifier: Apache-2.0
"""Attribute ncu per-SASS metrics (source page, --print-source sass) to CUDA
source lines using the cubin's line table (nvdisasm -g).
usage: python scripts/ncu_lines.py REPORT.ncu-rep CUBIN SYMBOL_SUBSTR [topN]"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, sym = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
syms = subprocess.run(["cuobjdump", "-symbols", cubin], capture_output=True, text=True).stdout
name = [l.split()[-1] for l in syms.splitlines() if sym in l and "$" not in l.split()[-1] and l.split()[0] == "STT_FUNC"][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
addr2line, cur, inside = {}, None, False
for l in dis.splitlines():
    if l.startswith(".text."):
        inside = l.strip().rstrip(":") == ".text." + name
        continue
    if not inside:
        continue
    if "//## File" in l:
        locs = re.findall(r'"([^"]+)", line (\d+)', l)
        # outermost call site (last in the inlining chain) unless --inner
        f, n = locs[0] if "--inner" in sys.argv else locs[-1]
        cur = f"{f.split('/')[-1]}:{n}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        addr2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ai, ie = h.index("Address"), h.index("Instructions Executed")
base = min(int(r[ai], 16) for r in rows[2:] if r[ai].startswith("0x"))
si = h.index("Warp Stall Sampling (All Samples)")
agg, stall = defaultdict(float), defaultdict(float)
tot = tots = 0.0
for r in rows[2:]:
    try:
        a = int(r[ai], 16) - base
    except ValueError:
        continue
    v = float(r[ie] or 0)
    s = float(r[si] or 0)
    ln = addr2line.get(a, "?")
    agg[ln] += v
    stall[ln] += s
    tot += v
    tots += s
src = {}
for ln in agg:
    f, n = ln.rsplit(":", 1) if ":" in ln else (ln, "0")
print(f"total warp-instructions {tot:.4g}, stall samples {tots:.4g}")
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / tot * 100:6.2f}% inst  {stall[ln] / max(tots, 1) * 100:6.2f}% stall  {ln}")
