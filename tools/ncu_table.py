#!/usr/bin/env python
"""Print a compact table of an ncu raw-page CSV export (one row per profiled launch):
time, DRAM read/write, FP64 pipe, warps active, registers and the top stall reasons.
usage: python tools/ncu_table.py raw.csv [label1,label2,...]"""
import csv
import io
import sys

rows = list(csv.reader(io.StringIO(open(sys.argv[1]).read())))
h, units, data = rows[0], rows[1], rows[2:]
labels = sys.argv[2].split(",") if len(sys.argv) > 2 else []
col = {c: h.index(c) for c in h}
def g(r, c):
    return r[col[c]] if c in col else ""
print("%-44s %9s %9s %9s %6s %6s %4s  %s" % ("kernel", "ms", "rd GB", "wr GB", "fp64%", "warps%", "regs", "top stalls"))
for i, r in enumerate(data):
    st = [(c, float(r[j])) for c, j in col.items() if c.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not c.endswith("_not_issued") and r[j] not in ("", "n/a")]
    tot = sum(v for _, v in st) or 1.0
    st.sort(key=lambda x: -x[1])
    stalls = " ".join("%s=%.0f%%" % (k.replace("smsp__pcsamp_warps_issue_stalled_", ""), 100 * v / tot) for k, v in st[:3])
    scale = {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}
    rd = float(g(r, "dram__bytes_read.sum") or 0) * scale.get(units[col["dram__bytes_read.sum"]], 1)
    wr = float(g(r, "dram__bytes_write.sum") or 0) * scale.get(units[col["dram__bytes_write.sum"]], 1)
    t = float(g(r, "gpu__time_duration.sum")) * (1e-3 if units[col["gpu__time_duration.sum"]] == "us" else 1)
    name = (labels[i] + ": " if i < len(labels) else "") + g(r, "Kernel Name")[:40]
    print("%-44s %9.4f %9.3f %9.3f %6.1f %6.1f %4s  %s" % (
        name[:44], t, rd, wr, float(g(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") or 0),
        float(g(r, "sm__warps_active.avg.pct_of_peak_sustained_active") or 0),
        g(r, "launch__registers_per_thread"), stalls))
