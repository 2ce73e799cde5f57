#!/bin/bash
# A/B: elements per tile (= threads per CTA) for the element kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for T in 256 128 64; do
  FEM_NVCC_FLAGS="-DFEM_TILE=$T" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/build_T$T.log 2>&1
  timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 > gpurun_out/bench_T$T.json 2> gpurun_out/bench_T$T.err
done
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
