#!/bin/bash
# ncu --set full of the bench step's kernels matching $K (default: the element kernels), raw +
# SASS source pages under gpurun_out/${TAG}_*
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-ps}; K=${K:-k_tile_pipe}; C=${C:-3}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"$K" -c $C -o gpurun_out/${T} -f python bench.py --profile-step > gpurun_out/${T}_ncu.log 2>&1
ncu -i gpurun_out/${T}.ncu-rep --page raw --csv > gpurun_out/${T}_raw.csv 2>/dev/null
for i in $(seq 0 $((C-1))); do ncu -i gpurun_out/${T}.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 2>/dev/null | gzip > gpurun_out/${T}_src$i.csv.gz; done
rm -f gpurun_out/${T}.ncu-rep; tail -2 gpurun_out/${T}_ncu.log
