#!/usr/bin/env python
"""DOF sweep ("vs DOFs" axis of the metric; BASELINE cfg 5 linear-scaling check, PAPER.md
Fig. 4 / P:331-339): per size, device time of energy / residual / HVP / sparse-tangent
assembly / SpMV and setup (pattern, coloring), CSV in the SPEC S:844 layout plus log-log
slopes.  L2 is flushed (256 MB write) before every timed call.

usage: python tools/sweep.py [out_prefix]   (run on a GPU box via gpurun)
"""
import csv
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fem_inputs as fi  # noqa: E402
from paper_2602_12365_b200 import build, fem  # noqa: E402

CASES = [("cfg5: 2D LE + periodic MPC", lambda n: fi.config_mesh(5, n=n), (70, 223, 706, 2235)),
         ("cfg2: 2D NH roller", lambda n: fi.config_mesh(2, n=n), (70, 223, 706, 2235)),
         ("cfg3: 3D NH roller (Kuhn)", lambda n: fi.config_mesh(3, n=n), (21, 46, 99, 150, 200))]


def main(prefix):
    build.build()
    flush = torch.empty(256 * 2 ** 20 // 8, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        return float(np.median(ts))

    rows, slopes = [], {}
    for name, make, sizes in CASES:
        per_op = {}
        for n in sizes:
            mesh = make(n)
            h = mesh.length / max(mesh.shape)
            z = torch.as_tensor(fi.lift(mesh, fi.generic_state(mesh, 5, eps=0.05, noise=0.01, h=h)),
                                device="cuda")
            v = torch.as_tensor(fi.random_direction(mesh.n_total, 4), device="cuda")
            p = fem.Problem(mesh)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            nnz = p.nnz()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            _, nc = p.color()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            vals = torch.empty(nnz, dtype=torch.float64, device="cuda")
            y = torch.empty(mesh.n_total, dtype=torch.float64, device="cuda")
            e = torch.empty(1, dtype=torch.float64, device="cuda")
            ops = {
                "energy": lambda: p.energy(z, out=e),
                "residual": lambda: p.residual(z, bc=True, out=y),
                "hvp": lambda: p.hvp(z, v, bc=True, out=y),
                "assemble_csr": lambda: p.assemble_csr(z, bc=True, out=vals),
                "assemble_jcomp": lambda: p.assemble_csr(z, bc=True, mode="batched", out=vals),
                "spmv": lambda: p.spmv(vals, v, out=y),
            }
            p.assemble_csr(z, bc=True, out=vals)
            res = {k: timed(f) for k, f in ops.items()}
            res["pattern"] = t1 - t0
            res["coloring"] = t2 - t1
            p.check()
            for op, t in res.items():
                rows.append({"problem": name, "mode": op, "n_dofs": mesh.n_total, "time_s": t,
                             "throughput_dofs_per_s": mesh.n_total / t, "n_colors": nc,
                             "status": "ok", "nnz": nnz, "gpus": 1, "impl": "b200-x1"})
                per_op.setdefault(op, []).append((mesh.n_total, t))
            del p, vals, y
            torch.cuda.empty_cache()
            print(name, n, mesh.n_total, {k: round(1e3 * t, 3) for k, t in res.items()}, flush=True)
        slopes[name] = {op: float(np.polyfit(np.log([a for a, _ in pts]), np.log([b for _, b in pts]), 1)[0])
                        for op, pts in per_op.items()}
        # asymptotic slope over the two largest sizes (launch overhead dominates small ones)
        slopes[name + " (two largest)"] = {
            op: float(np.log(pts[-1][1] / pts[-2][1]) / np.log(pts[-1][0] / pts[-2][0]))
            for op, pts in per_op.items()}
    with open(prefix + "_sweep.csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
    json.dump({"loglog_slope_time_vs_dofs": slopes,
               "note": "slope of log(time) vs log(N_dofs) over the sizes; 1.0 = O(N)"},
              open(prefix + "_sweep_slopes.json", "w"), indent=1)
    print(json.dumps(slopes, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "r01"))
