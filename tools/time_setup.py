"""Time the setup phases (create, pattern, coloring) of a BASELINE config twice."""
import sys
import time

import torch

sys.path.insert(0, ".")
import fem_inputs as fi  # noqa: E402
from paper_2602_12365_b200 import build, fem  # noqa: E402

build.build()
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mesh = fi.config_mesh(cfg)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = fem.Problem(mesh)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    nnz = p.nnz()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    _, nc = p.color()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms  pattern {1e3*(t2-t1):.1f} ms  "
          f"coloring {1e3*(t3-t2):.1f} ms  nnz {nnz} colors {nc}", flush=True)
    del p
