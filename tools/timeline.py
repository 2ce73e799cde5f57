#!/usr/bin/env python
"""GPU timeline of CG iterations (CUPTI kernel activity via torch.profiler; nsys is not in the
image): matrix-free (HVP) and CSR CG on the bench workload, with and without CUDA graphs.
Writes profiles/<tag>_cg_timeline.csv (per kernel: start / duration relative to the first
kernel) and a summary JSON (per iteration: kernel time, idle gap, launches).

usage: python tools/timeline.py [--tag r02] [--config 3] [--iters 16]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2602_12365_b200 import fem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tag", default="r02")
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--iters", type=int, default=16)
a = ap.parse_args()
mesh, name, z, v = bench.workload(a.config, a.n)
prob = fem.Problem(mesh)
zt = torch.as_tensor(z, device="cuda")
b = torch.as_tensor(v, device="cuda").clone()
b[torch.as_tensor(mesh.dirichlet_dofs.astype(np.int64), device="cuda")] = 0.0
vals = prob.assemble_csr(zt, bc=True)
rows, summary = [], {}
for label, op, env in (("hvp_graph", 0, None), ("hvp_direct", 0, "1"), ("csr_graph", 1, None),
                       ("csr_direct", 1, "1")):
    if env:
        os.environ["FEM_NO_GRAPHS"] = env
    else:
        os.environ.pop("FEM_NO_GRAPHS", None)
    prob.cg_solve(b, z=zt, vals=vals, op=op, rtol=1e-30, max_iter=4, check_every=4, raise_on_fail=False)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        prob.cg_solve(b, z=zt, vals=vals, op=op, rtol=1e-30, max_iter=a.iters, check_every=a.iters,
                      raise_on_fail=False)
        torch.cuda.synchronize()
    ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"],
                key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    busy, prev_end, gaps = 0.0, None, 0.0
    for e in ev:
        s, t = e.time_range.start, e.time_range.end
        rows.append((label, e.name[:70], (s - t0) / 1e3, (t - s) / 1e3))
        busy += t - s
        if prev_end is not None and s > prev_end:
            gaps += s - prev_end
        prev_end = max(prev_end or t, t)
    span = prev_end - t0
    summary[label] = {"iters": a.iters, "span_ms": span / 1e3, "kernel_ms": busy / 1e3,
                      "idle_ms": gaps / 1e3, "ms_per_iter": span / 1e3 / a.iters,
                      "launches": len(ev), "launches_per_iter": len(ev) / a.iters}
os.environ.pop("FEM_NO_GRAPHS", None)
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", f"{a.tag}_cg_timeline.csv"), "w") as f:
    f.write("run,kernel,start_ms,duration_ms\n")
    for r in rows:
        f.write(f"{r[0]},\"{r[1]}\",{r[2]:.4f},{r[3]:.4f}\n")
summary["workload"] = name
json.dump(summary, open(os.path.join(ROOT, "profiles", f"{a.tag}_cg_timeline_summary.json"), "w"), indent=1)
print(json.dumps(summary, indent=1))
