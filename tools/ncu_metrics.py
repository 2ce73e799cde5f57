#!/usr/bin/env python
"""Key metrics per kernel from an ncu raw CSV page: usage ncu_metrics.py raw.csv [more...]"""
import csv
import sys

KEYS = [("gpu__time_duration.sum", "ms"), ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%"),
        ("sm__inst_executed.avg.per_cycle_active", "ipc"), ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"), ("launch__registers_per_thread", "regs"),
        ("dram__bytes_read.sum", "dramR"), ("dram__bytes_write.sum", "dramW"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
        ("smsp__inst_executed.sum", "inst")]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:40]
        out = []
        for k, lab in KEYS:
            if k in h:
                out.append(f"{lab}={r[h.index(k)]}{u[h.index(k)] if lab.startswith('dram') else ''}")
        st = [(h[i][len('smsp__pcsamp_warps_issue_stalled_'):], float(r[i])) for i in range(len(h))
              if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")
              and r[i] not in ("", "n/a")]
        tot = sum(v for _, v in st) or 1
        st.sort(key=lambda x: -x[1])
        print(name, " ".join(out), " | ", " ".join(f"{k}={100*v/tot:.0f}%" for k, v in st[:6]))
