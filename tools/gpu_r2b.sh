#!/bin/bash
# S-variant / colored-scatter evidence: tests, bench (ab), ncu of the variants.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-r2b}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -30 gpurun_out/${T}_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${TESTS:-residual_hvp_modes or full_size_sampled or delaunay_1e5}" > gpurun_out/${T}_tests.log 2>&1
tail -4 gpurun_out/${T}_tests.log
timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python - "$T" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/{t}_bench.json").read().strip().splitlines()[-1])
    print("value", d["value"], "step ms", d["ms_per_step"])
    for k, v in d["phases"].items(): print(f"  {k:9s} {v['ms']:.3f} ms")
    print("ab", json.dumps(d.get("ab")))
except Exception as e:
    print("bench failed", e); print(open(f"gpurun_out/{t}_bench.err").read()[-3000:])
PY
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_tile_pipe" -c 4 \
  -o gpurun_out/${T}_ncu_tiles -f python tools/profile_variants.py --variants hvp,hvp_s,res,res_s > gpurun_out/${T}_ncu_tiles.log 2>&1
tail -2 gpurun_out/${T}_ncu_tiles.log
ncu -i gpurun_out/${T}_ncu_tiles.ncu-rep --page raw --csv > gpurun_out/${T}_ncu_tiles_raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.avg.per_cycle_active,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum \
  --clock-control none --profile-from-start off -k regex:"k_elem|k_tile_pipe" --csv --log-file gpurun_out/${T}_ncu_col.csv \
  python tools/profile_variants.py --variants hvp,hvp_col,hvp_atomic,res,res_col > gpurun_out/${T}_ncu_col.log 2>&1
tail -2 gpurun_out/${T}_ncu_col.log
