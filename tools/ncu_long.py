#!/usr/bin/env python
"""Aggregate an `ncu --metrics ... --csv` launch list (long format) per consecutive run of the
same kernel: launches, total time, DRAM bytes, L2 RED/atomic sectors, time-weighted FP64 pipe."""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]
ik, im, iv, iu, iid = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
SC = {"ms": 1e-3, "msecond": 1e-3, "us": 1e-6, "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9,
      "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
per = collections.OrderedDict()
for r in rows[1:]:
    if len(r) < len(h):
        continue
    d = per.setdefault(r[iid], {"name": r[ik]})
    d[r[im]] = float(r[iv].replace(",", "")) * SC.get(r[iu], 1.0)
groups = []
for d in per.values():
    if groups and groups[-1]["name"] == d["name"] and "k_elem" in d["name"]:
        g = groups[-1]
    else:
        g = {"name": d["name"], "n": 0, "t": 0.0, "dr": 0.0, "dw": 0.0, "red": 0.0, "atom": 0.0, "fp": 0.0}
        groups.append(g)
    t = d.get("gpu__time_duration.sum", 0.0)
    g["n"] += 1
    g["t"] += t
    g["dr"] += d.get("dram__bytes_read.sum", 0.0)
    g["dw"] += d.get("dram__bytes_write.sum", 0.0)
    g["red"] += d.get("lts__t_sectors_op_red.sum", 0.0)
    g["atom"] += d.get("lts__t_sectors_op_atom.sum", 0.0)
    g["fp"] += d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0) * t
print("kernel,launches,ms,dram_read_GB,dram_write_GB,GB_per_s,l2_red_sectors_M,l2_atom_sectors_M,fp64_pipe_pct")
for g in groups:
    print(f"\"{g['name'][:60]}\",{g['n']},{g['t'] * 1e3:.4f},{g['dr'] / 1e9:.4f},{g['dw'] / 1e9:.4f},"
          f"{(g['dr'] + g['dw']) / max(g['t'], 1e-12) / 1e9:.0f},{g['red'] / 1e6:.2f},{g['atom'] / 1e6:.2f},"
          f"{g['fp'] / max(g['t'], 1e-12):.1f}")
