#!/bin/bash
# Knob re-check on the G8 HVP (device-timed energy / residual / HVP).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for FL in "-DFEM_ISSUE_NODE=0" "" "-DFEM_ISSUE_NODE=0" ""; do
  FEM_NVCC_FLAGS="$FL" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/r2ab_b.log 2>&1 || { echo "build failed $FL"; continue; }
  echo "[$FL] $(timeout 600 python tools/time_ops.py 2>&1 | tail -1)"
done
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
