#!/bin/bash
# A/B of compile-time tile parameters: FEM_TILE (elements per tile) x FEM_PIPE_MINB.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for V in "256 3" "128 3" "128 4" "256 2"; do
  set -- $V
  FEM_NVCC_FLAGS="-DFEM_TILE=$1 -DFEM_PIPE_MINB=$2" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/build_t$1_m$2.log 2>&1
  timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 > gpurun_out/bench_t$1_m$2.json 2> gpurun_out/bench_t$1_m$2.err
done
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
