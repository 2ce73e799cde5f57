#!/bin/bash
# Node-tile assembly micro-changes: per-node staging (FEM_RT_ISSUE_NODE), unrolled diagonal
# sums (FEM_RT_DIAG_UNROLL), arithmetic pair index; parity of the assembly tests, then A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1 || { tail -20 gpurun_out/r2i_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "assembly or rows or row_ or spmv" > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2i_tests.log
bash tools/ab_flags.sh "" "-DFEM_RT_ISSUE_NODE=0" "-DFEM_RT_DIAG_UNROLL=0" "-DFEM_RT_ISSUE_NODE=0 -DFEM_RT_DIAG_UNROLL=0" ""
