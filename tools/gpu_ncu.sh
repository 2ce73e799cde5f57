#!/bin/bash
# ncu --set full capture of the kernels matching $NCU_KERNELS over one bench step
# (--profile-step), exported to CSV in gpurun_out/ (raw + source pages).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=${TAG:-cap}
timeout ${NCU_TIMEOUT:-1200} ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"${NCU_KERNELS}" -c ${NCU_COUNT:-4} -o gpurun_out/$TAG -f \
   python bench.py --profile-step ${BENCH_ARGS:-} > gpurun_out/${TAG}.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
tail -3 gpurun_out/${TAG}.log
