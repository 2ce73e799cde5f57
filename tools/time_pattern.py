import time, torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
import fem_inputs as fi
from paper_2602_12365_b200 import build, fem
build.build()
torch.cuda.set_device(0)
mesh = fi.config_mesh(3)
for rep in range(2):
    p = fem.Problem(mesh)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    nnz = p.nnz(); torch.cuda.synchronize(); t1 = time.perf_counter()
    _, nc = p.color(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(rep, "pattern", round((t1-t0)*1e3, 1), "color", round((t2-t1)*1e3, 1), flush=True)
    del p
