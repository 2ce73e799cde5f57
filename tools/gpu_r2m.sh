#!/bin/bash
# Phase-2 long-node split (FEM_P2_LSPLIT threshold; 0 = off): parity of the element-operator
# tests, then the quick-bench A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2m_build.log 2>&1 || { tail -20 gpurun_out/r2m_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -k "energy or residual or hvp or linearized or newton or cg or full_size or delaunay or cfg4" > gpurun_out/r2m_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2m_tests.log
bash tools/ab_flags.sh "" "-DFEM_P2_LSPLIT=0" "-DFEM_P2_LSPLIT=8" "-DFEM_P2_LSPLIT=16" "" "-DFEM_P2_LSPLIT=0"
