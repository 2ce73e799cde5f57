#!/bin/bash
# Full ncu capture (source counters) of one cfg 3 node-tile assembly launch (default records).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2h_build.log 2>&1 || { tail -20 gpurun_out/r2h_build.log; exit 1; }
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_rows_tile --launch-skip 1 -c 1 -o gpurun_out/r2h_rows -f python tools/prof_rows.py > gpurun_out/r2h_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r2h_ncu.log; ls -la gpurun_out/r2h_rows.ncu-rep
