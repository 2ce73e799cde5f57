#!/bin/bash
# Re-run the phase-2 variants on the round-2 kernels (device-timed energy / residual / HVP).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for FL in "" "-DFEM_P2_G8=1" "-DFEM_P2_BAL=1" "-DFEM_P2_PAIR=1" "-DFEM_P2_NM=1" ""; do
  FEM_NVCC_FLAGS="$FL" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/r2v_build.log 2>&1 || { echo "build failed $FL"; tail -3 gpurun_out/r2v_build.log; continue; }
  echo "[$FL] $(timeout 600 python tools/time_ops.py 2>&1 | tail -1)"
done
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
