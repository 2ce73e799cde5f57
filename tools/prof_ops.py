#!/usr/bin/env python
"""cfg 3 element operators after a warm-up (energy, residual, HVP with BC): the launches ncu
captures with `-k regex:k_tile_pipe` (tools/gpu_r2j.sh)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fem_inputs as fi  # noqa: E402
from paper_2602_12365_b200 import fem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 150
mesh = fi.config_mesh(3, n=n)
prob = fem.Problem(mesh)
z = torch.as_tensor(fi.lift(mesh, fi.generic_state(mesh, 5)), device="cuda")
v = torch.as_tensor(fi.random_direction(mesh.n_total, 6), device="cuda")
for _ in range(2):
    prob.energy(z)
    prob.residual(z, bc=True)
    prob.hvp(z, v, bc=True)
torch.cuda.synchronize()
print("ok")
