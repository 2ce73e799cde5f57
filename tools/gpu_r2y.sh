#!/bin/bash
# End-of-session ncu evidence on the final kernels: launch list of one bench step and the
# --set full capture of the step kernels (CSV exports), the cfg 4 strong P=1 line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=r02
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/${T}_launches.csv python bench.py --profile-step > gpurun_out/${T}_ncu_list.log 2>&1; echo "list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"k_tile_pipe|k_rows_tile|k_spmv" -c 5 -o gpurun_out/${T}_prof_full -f \
   python bench.py --profile-step > gpurun_out/${T}_ncu_full.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/${T}_prof_full.ncu-rep --page raw --csv > gpurun_out/${T}_prof_full_raw.csv 2>/dev/null
ncu -i gpurun_out/${T}_prof_full.ncu-rep --page source --csv --print-source sass --launch-skip 2 --launch-count 1 2>/dev/null > gpurun_out/${T}_hvp_src.csv
rm -f gpurun_out/${T}_prof_full.ncu-rep
timeout 900 python bench.py --scaling strong --no-cpu-baseline --steps 5 > gpurun_out/${T}_strong.json 2> gpurun_out/${T}_strong.err; echo "strong rc=$?"
