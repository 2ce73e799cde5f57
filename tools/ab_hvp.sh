#!/bin/bash
# A/B of the tile kernel variants (compile-time flags), quick bench each.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for V in "0 3" "1 3" "0 2" "0 4"; do
  set -- $V
  FEM_NVCC_FLAGS="-DFEM_PHASE2_SPLIT=$1 -DFEM_PIPE_MINB=$2" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/build_h$1_$2.log 2>&1
  timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 > gpurun_out/bench_h$1_$2.json 2> gpurun_out/bench_h$1_$2.err
done
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
