#!/bin/bash
# One gpurun session: parity tests, bench, ncu launch list and a full capture of the
# element kernels.  Outputs land in gpurun_out/ (scratch; summaries go to profiles/).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
MODE=${1:-all}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [[ $MODE == all || $MODE == tests ]]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/gpu_tests.log 2>&1
  tail -5 gpurun_out/gpu_tests.log
fi
if [[ $MODE == all || $MODE == bench ]]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
  tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
fi
if [[ $MODE == all || $MODE == ncu ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches.csv python bench.py --profile-step > gpurun_out/ncu_list.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on \
     -k regex:"${NCU_KERNELS:-k_tile_elem|k_colored_hvp|k_decompress|k_spmv|k_rows_gather}" -c ${NCU_COUNT:-6} \
     -o gpurun_out/prof_full -f python bench.py --profile-step > gpurun_out/ncu_full.log 2>&1
  tail -3 gpurun_out/ncu_full.log
fi
