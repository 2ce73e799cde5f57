#!/bin/bash
# Full ncu captures (source counters) of the cfg 3 energy, residual and HVP tile kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1 || { tail -20 gpurun_out/r2j_build.log; exit 1; }
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_tile_pipe --launch-skip 3 -c 3 -o gpurun_out/r2j_ops -f python tools/prof_ops.py > gpurun_out/r2j_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r2j_ncu.log; ls -la gpurun_out/r2j_ops.ncu-rep
