#!/bin/bash
# Residual on the decoupled (mbarrier) pipeline (FEM_RES_DEC) A/B on the round-2 kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2l_build.log 2>&1 || { tail -20 gpurun_out/r2l_build.log; exit 1; }
bash tools/ab_flags.sh "-DFEM_RES_DEC=1" "" "-DFEM_RES_DEC=1 -DFEM_RES_MINB=2" ""
