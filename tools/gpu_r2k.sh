#!/bin/bash
# HVP metadata depth (FEM_META_BUFS 3 / 4) A/B with parity of the HVP tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2k_build.log 2>&1 || { tail -20 gpurun_out/r2k_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "hvp or linearized or newton" > gpurun_out/r2k_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2k_tests.log
bash tools/ab_flags.sh "-DFEM_META_BUFS=4" "-DFEM_META_BUFS=3" "-DFEM_META_BUFS=4" "-DFEM_META_BUFS=3"
