#!/bin/bash
# A/B: fused row-pull assembly register budget (FEM_ROWS_MINB CTAs/SM).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for MB in 4 5 6; do
  FEM_NVCC_FLAGS="-DFEM_ROWS_MINB=$MB" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/build_r$MB.log 2>&1
  timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 > gpurun_out/bench_r$MB.json 2> gpurun_out/bench_r$MB.err
done
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
