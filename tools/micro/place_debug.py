import os, sys, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import fem_inputs as fi
from paper_2602_12365_b200 import fem, build
build.build()
mesh = fi.config_mesh(3, n=60)
prob = fem.Problem(mesh)
z = torch.as_tensor(fi.lift(mesh, fi.generic_state(mesh, 5)), device="cuda")
prob.assemble_csr(z, bc=True)
torch.cuda.synchronize(); print("ok")
