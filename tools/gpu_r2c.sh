#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-r2c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -30 gpurun_out/${T}_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${TESTS:-residual_hvp_modes or full_size_sampled}" > gpurun_out/${T}_tests.log 2>&1
tail -4 gpurun_out/${T}_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum \
  --clock-control none --profile-from-start off -k regex:"k_elem|k_tile_pipe" --csv --log-file gpurun_out/${T}_ncu_tcol.csv \
  python tools/profile_variants.py --variants hvp,hvp_tcol,res,res_tcol > gpurun_out/${T}_ncu_tcol.log 2>&1
python tools/ncu_long.py gpurun_out/${T}_ncu_tcol.csv
python - <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
import bench
from paper_2602_12365_b200 import fem
mesh, name, z, v = bench.workload(3, None)
p = fem.Problem(mesh)
zt, vt = torch.as_tensor(z, device="cuda"), torch.as_tensor(v, device="cuda")
y = torch.empty_like(zt)
for f in (0, fem.TILE_COLORED, fem.DETERMINISTIC):
    p.hvp(zt, vt, bc=True, out=y, flags=f); p.residual(zt, bc=True, out=y, flags=f)
    torch.cuda.synchronize()
    for op in ("hvp", "res"):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            p.hvp(zt, vt, bc=True, out=y, flags=f) if op == "hvp" else p.residual(zt, bc=True, out=y, flags=f)
        b.record(); torch.cuda.synchronize()
        print(f"flags={f} {op} {a.elapsed_time(b)/10:.4f} ms")
print("tile colors", len(p._h and []) if False else "")
PY
