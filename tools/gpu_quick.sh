#!/bin/bash
# quick perf check: build, one bench (no solves / cpu baseline), ncu of the named kernels
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 ${BENCH_ARGS:-} > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
if [[ -n "${NCU_KERNELS:-}" ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$NCU_KERNELS" -c ${NCU_COUNT:-2} \
     -o gpurun_out/prof_quick -f python bench.py --profile-step ${BENCH_ARGS:-} > gpurun_out/ncu_quick.log 2>&1
fi
