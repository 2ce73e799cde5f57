#!/usr/bin/env python
"""One cfg 3 sparse-tangent assembly (node tiles) after a warm-up call: the launch ncu
captures with `-k regex:k_rows_tile --launch-skip 1 -c 1` (tools/gpu_r2g.sh)."""
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
prob.sparsity()
for _ in range(2):
    prob.assemble_csr(z, bc=True)
torch.cuda.synchronize()
print("ok")
