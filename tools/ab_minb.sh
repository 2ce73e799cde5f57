#!/bin/bash
# A/B: persistent tile kernel with 3 vs 2 CTAs/SM register budget (quick bench each).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for MB in 3 2; do
  FEM_NVCC_FLAGS="-DFEM_PIPE_MINB=$MB" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/build_$MB.log 2>&1
  timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 > gpurun_out/bench_minb$MB.json 2> gpurun_out/bench_minb$MB.err
done
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
