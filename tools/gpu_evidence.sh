#!/bin/bash
# Round evidence in one call: smoke, full bench (default flags), reference arm, ncu launch
# list of one step, ncu --set full of the step's main kernels (CSV exports), all under
# gpurun_out/ (summaries copied to profiles/ by hand).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/launches.csv python bench.py --profile-step > gpurun_out/ncu_list.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"k_tile_pipe|k_rows_tile|k_spmv" -c 5 -o gpurun_out/prof_full -f \
   python bench.py --profile-step > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/prof_full.ncu-rep --page raw --csv > gpurun_out/prof_full_raw.csv 2>/dev/null
tail -2 gpurun_out/smoke.log; tail -c 400 gpurun_out/bench_full.json
