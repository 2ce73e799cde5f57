#!/usr/bin/env python
"""One call of each residual / HVP variant on the bench workload inside a profiler range, for
`ncu --profile-from-start off` (kernel-choice evidence).

usage: python tools/profile_variants.py [--config 3] [--variants hvp,hvp_s,hvp_col,...]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_12365_b200 import fem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--variants", default="hvp,hvp_s,hvp_col,res,res_s,res_col")
a = ap.parse_args()
mesh, name, z, v = bench.workload(a.config, a.n)
prob = fem.Problem(mesh)
zt = torch.as_tensor(z, device="cuda")
vt = torch.as_tensor(v, device="cuda")
y = torch.empty_like(zt)
calls = {
    "hvp": lambda: prob.hvp(zt, vt, bc=True, out=y),
    "hvp_s": lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.STREAM_GEOM),
    "hvp_col": lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.COLORED_SCATTER),
    "hvp_atomic": lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.BASELINE_SCATTER),
    "hvp_tcol": lambda: prob.hvp(zt, vt, bc=True, out=y, flags=fem.TILE_COLORED),
    "res": lambda: prob.residual(zt, bc=True, out=y),
    "res_tcol": lambda: prob.residual(zt, bc=True, out=y, flags=fem.TILE_COLORED),
    "res_s": lambda: prob.residual(zt, bc=True, out=y, flags=fem.STREAM_GEOM),
    "res_col": lambda: prob.residual(zt, bc=True, out=y, flags=fem.COLORED_SCATTER),
    "hvp_lin": lambda: (prob.hvp(zt, vt, bc=True, out=y, flags=fem.LINEARIZED)),
    "energy": lambda: prob.energy(zt),
    "assemble_col": lambda: prob.assemble_csr(zt, bc=True, mode="colored"),
    "assemble": lambda: prob.assemble_csr(zt, bc=True),
}
sel = a.variants.split(",")
prob.linearize(zt)
for k in sel:          # warm: lazy setup (geometry stream, element colors, pattern)
    calls[k]()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for k in sel:
    calls[k]()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
prob.check()
print("profiled", sel)
