import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import bench
from paper_2602_12365_b200 import fem
mesh, name, z, v = bench.workload(2, None)
prob = fem.Problem(mesh)
zt = torch.as_tensor(z, device="cuda")
b0 = torch.as_tensor(v, device="cuda").clone()
b0[torch.as_tensor(mesh.dirichlet_dofs.astype(np.int64), device="cuda")] = 0.0
vals = prob.assemble_csr(zt, bc=True)
def run(label, op=0):
    torch.cuda.synchronize()
    t = time.perf_counter()
    _, info = prob.cg_solve(b0, z=zt, vals=vals, op=op, rtol=1e-30, max_iter=256, check_every=32, raise_on_fail=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{label}: op={op} iters={info['iters']} {1e3*dt/max(info['iters'],1):.4f} ms/iter converged={info['converged']}", flush=True)
run("first"); run("second"); run("csr", 1)
os.environ["FEM_NO_GRAPHS"] = "1"; run("nographs"); os.environ.pop("FEM_NO_GRAPHS")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    prob.hvp(zt, zt, bc=True); torch.cuda.synchronize()
run("after_profiler"); run("after_profiler_csr", 1)
