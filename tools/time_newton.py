#!/usr/bin/env python
"""Wall time of the cfg 3 Newton solves (matrix-free / CSR, fixed / Eisenstat-Walker inner
tolerances) as bench.py runs them, for A/Bs of the solver path."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fem_inputs as fi  # noqa: E402
from paper_2602_12365_b200 import build, fem  # noqa: E402

build.build()
mesh = fi.config_mesh(3, n=int(sys.argv[1]) if len(sys.argv) > 1 else 150)
prob = fem.Problem(mesh)
eps = float(mesh.dirichlet_vals.max()) / mesh.length
z0 = torch.as_tensor(fi.lift(mesh, fi.affine_field(mesh, np.diag([eps, 0.0, 0.0]))), device="cuda")
prob.nnz()
prob.color()
out = []
for op, jac, forcing in ((0, False, 0.0), (1, True, 0.0), (0, False, 0.9), (1, True, 0.9)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    z, info = prob.newton_solve(z0, op=op, jacobi=jac, cg_rtol=1e-8, rtol=1e-10, atol=1e-14,
                                check_every=16, raise_on_fail=False, forcing=forcing)
    torch.cuda.synchronize()
    out.append(f"op={op} forcing={forcing}: {time.perf_counter() - t0:.3f} s ({info['iters']} it, {info['cg_iters']} CG)")
print(" | ".join(out))
