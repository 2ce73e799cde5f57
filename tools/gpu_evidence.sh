#!/bin/bash
# Round evidence in one call (TAG names the outputs): smoke, full bench (default flags), the
# reference arm, cfg4 strong P=1, ncu launch list of one step, ncu --set full of the step's
# main kernels and of the residual / HVP variants (CSV exports), under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-ev}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 900 python bench.py --scaling strong --no-cpu-baseline --steps 5 > gpurun_out/${T}_strong.json 2> gpurun_out/${T}_strong.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/${T}_launches.csv python bench.py --profile-step > gpurun_out/${T}_ncu_list.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"k_tile_pipe|k_rows_tile|k_spmv" -c 5 -o gpurun_out/${T}_prof_full -f \
   python bench.py --profile-step > gpurun_out/${T}_ncu_full.log 2>&1
ncu -i gpurun_out/${T}_prof_full.ncu-rep --page raw --csv > gpurun_out/${T}_prof_full_raw.csv 2>/dev/null
for i in 0 1 2 3 4; do
  ncu -i gpurun_out/${T}_prof_full.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 2>/dev/null | gzip > gpurun_out/${T}_prof_full_src$i.csv.gz
done
mkdir -p /tmp/ncu_keep && mv gpurun_out/${T}_prof_full.ncu-rep /tmp/ncu_keep/   # > 64 MiB with the rest
timeout 1200 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:"k_tile_pipe|k_rows_fused|k_elem_ctx|k_rows_tile" -c 12 -o gpurun_out/${T}_prof_var -f \
   python tools/profile_variants.py --variants hvp,hvp_lin,hvp_s,res,res_s,assemble_col > gpurun_out/${T}_ncu_var.log 2>&1
ncu -i gpurun_out/${T}_prof_var.ncu-rep --page raw --csv > gpurun_out/${T}_prof_var_raw.csv 2>/dev/null
mv gpurun_out/${T}_prof_var.ncu-rep /tmp/ncu_keep/
tail -2 gpurun_out/${T}_smoke.log; tail -c 300 gpurun_out/${T}_bench.json; echo; tail -c 200 gpurun_out/${T}_strong.json
