# SPDX-License-Identifier: Apache-2.0
"""Summarise an ncu report (--set full) into the text kept under profiles/.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [units_per_launch bytes_per_unit] > profiles/....txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TSCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def num(s):
    return float(s.replace(",", ""))


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        print(f"kernel: {vals[hdr.index('Kernel Name')]}")
        got = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:58s} {vals[i]:>20s} {units[i]}")
                got[k] = (vals[i], units[i])
        if len(sys.argv) >= 4 and "dram__bytes_read.sum" in got:
            n, per = float(sys.argv[2]), float(sys.argv[3])
            rd = num(got["dram__bytes_read.sum"][0]) * SCALE[got["dram__bytes_read.sum"][1]]
            wr = num(got["dram__bytes_write.sum"][0]) * SCALE[got["dram__bytes_write.sum"][1]]
            t_s = num(got["gpu__time_duration.sum"][0]) * TSCALE.get(got["gpu__time_duration.sum"][1], 1e-9)
            print(f"  units/launch {n:.0f}, algorithmic bytes/unit {per:.0f} -> algorithmic {n * per / 1e9:.4f} GB, "
                  f"dram traffic {(rd + wr) / 1e9:.4f} GB ({(rd + wr) / (n * per):.3f}x algorithmic), "
                  f"algorithmic GB/s under ncu (cold, serialised) {n * per / t_s / 1e9:.1f}")


if __name__ == "__main__":
    main()
