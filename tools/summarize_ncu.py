#!/usr/bin/env python
"""Summarise an ncu --set full report and an ncu launch list into profiles/<tag>_*.

usage: python tools/summarize_ncu.py <tag> <prof.ncu-rep | raw.csv> <launches.csv>
Writes profiles/<tag>_ncu_kernels.csv (per captured kernel: time, DRAM traffic, pipe use,
occupancy, stall mix), profiles/<tag>_launches.csv (the launch list, kernel name + duration),
profiles/<tag>_step_shares.csv (one bench step's kernels with their share of the step) and
profiles/ncu_traffic.json (DRAM bytes per launch of the step's kernels, read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PHASE_OF = {"k_tile_pipe<3, 1, 0": "energy", "k_tile_pipe<3, 1, 1": "residual",
            "k_tile_pipe<3, 1, 2": "hvp", "k_rows_fused": "assemble", "k_rows_pull": "assemble", "k_rows_tile": "assemble", "k_elem_ctx": "assemble",
            "k_spmv": "spmv"}


def raw(rep):
    """the raw page of an ncu report (.ncu-rep) or its CSV export (ncu -i … --page raw --csv)"""
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def main(tag, rep, launches):
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    h, units, rows = raw(rep)
    cols = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]
    idx = [h.index(c) for c in cols if c in h]
    traffic = {}
    with open(os.path.join(prof, f"{tag}_ncu_kernels.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow([h[i] for i in idx] + ["top stalls"])
        w.writerow([units[i] for i in idx] + [""])
        for row in rows:
            st = [(h[i], float(row[i])) for i in range(len(h))
                  if h[i].startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h[i].endswith("_not_issued") and row[i] not in ("", "n/a")]
            tot = sum(v for _, v in st) or 1.0
            st.sort(key=lambda x: -x[1])
            stalls = " ".join("%s=%.0f%%" % (k.replace("smsp__pcsamp_warps_issue_stalled_", ""),
                                             100 * v / tot) for k, v in st[:4])
            w.writerow([row[i][:70] for i in idx] + [stalls])
            name = row[h.index("Kernel Name")]
            gb = float(row[h.index("dram__bytes_read.sum")]) + float(row[h.index("dram__bytes_write.sum")])
            unit = units[h.index("dram__bytes_read.sum")]
            scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)
            for key, phase in PHASE_OF.items():
                if key in name:
                    traffic.setdefault(phase, 0.0)
                    traffic[phase] += gb * scale
    json.dump({"source": f"profiles/{tag}_ncu_kernels.csv (ncu --set full, one launch each)",
               "dram_bytes_per_launch": traffic}, open(os.path.join(prof, "ncu_traffic.json"), "w"),
              indent=1)
    # launch list
    lines = [l for l in open(launches) if not l.startswith("==")]
    r = list(csv.reader(io.StringIO("".join(lines))))
    hh = r[0]
    kn, val = hh.index("Kernel Name"), hh.index("Metric Value")
    seq = [(x[kn], float(x[val])) for x in r[1:] if len(x) > val]
    with open(os.path.join(prof, f"{tag}_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "gpu__time_duration_ns"])
        for k, v in seq:
            w.writerow([k[:100], int(v)])
    # launch list taken with --profile-from-start off around exactly one bench step
    step = seq
    tot = sum(v for _, v in step) or 1.0
    with open(os.path.join(prof, f"{tag}_step_shares.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "ns", "share_of_step"])
        for k, v in step:
            w.writerow([k[:100], int(v), "%.4f" % (v / tot)])
    print(f"wrote profiles/{tag}_*.csv and profiles/ncu_traffic.json; step kernels: {len(step)}")


if __name__ == "__main__":
    main(*sys.argv[1:4])
