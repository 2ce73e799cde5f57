#!/usr/bin/env python
"""Device time (CUDA events, median of 10 after 3 warm-ups) of the default-mode cfg 3 energy,
residual and HVP — a minimal A/B timer for compile-time experiments that break other modes."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fem_inputs as fi  # noqa: E402
from paper_2602_12365_b200 import build, fem  # noqa: E402

build.build()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 150
mesh = fi.config_mesh(3, n=n)
prob = fem.Problem(mesh)
z = torch.as_tensor(fi.lift(mesh, fi.generic_state(mesh, 5)), device="cuda")
v = torch.as_tensor(fi.random_direction(mesh.n_total, 6), device="cuda")
out = {}
for name, fn in (("energy", lambda: prob.energy(z)), ("residual", lambda: prob.residual(z, bc=True)),
                 ("hvp", lambda: prob.hvp(z, v, bc=True))):
    ts = []
    for k in range(13):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if k >= 3:
            ts.append(a.elapsed_time(b))
    out[name] = float(np.median(ts))
y = prob.hvp(z, v, bc=True)
print(" ".join(f"{k}={v:.3f}" for k, v in out.items()), "| hvp checksum", float(y.abs().sum()))
