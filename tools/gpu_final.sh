#!/bin/bash
# Round-end evidence in one call: full -m gpu suite + round evidence (gpu_round.sh), the
# compute-sanitizer pass, the unstructured (cfg 6) and cfg 2 bench lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-r02}
TAG=$T bash tools/gpu_round.sh
TAG=${T}_san bash tools/sanitize.sh > gpurun_out/${T}_sanitizer.txt 2>&1
timeout 1500 python bench.py --config 6 --no-solve --no-cpu-baseline --steps 10 > gpurun_out/${T}_bench_delaunay.json 2> gpurun_out/${T}_bench_delaunay.err
timeout 900 python bench.py --config 2 --steps 20 > gpurun_out/${T}_bench_cfg2.json 2> gpurun_out/${T}_bench_cfg2.err
tail -c 300 gpurun_out/${T}_bench_delaunay.json; echo; tail -c 300 gpurun_out/${T}_bench_cfg2.json; echo; cat gpurun_out/${T}_sanitizer.txt
