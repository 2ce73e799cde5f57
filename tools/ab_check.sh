#!/bin/bash
# A/B over compile-time variants with gpu_check.sh (no tests): one quick bench per argument
# (a set of nvcc -D flags), phases and A/B entries printed; then the default build restored.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
i=0
for FL in "$@"; do
  i=$((i+1))
  echo "=== [$FL]"
  TAG=ab$i TESTS=0 FEM_NVCC_FLAGS="$FL -DFEM_AB_TAG=$i" bash tools/gpu_check.sh 2>&1 | grep -v "^$"
done
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
