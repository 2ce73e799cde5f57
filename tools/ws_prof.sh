cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
FEM_NVCC_FLAGS="-DFEM_WS=1 ${WSF:-}" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/wsp_build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_tile_ws" -c 2 -o gpurun_out/wsp -f python bench.py --profile-step > gpurun_out/wsp_ncu.log 2>&1
ncu -i gpurun_out/wsp.ncu-rep --page raw --csv > gpurun_out/wsp_raw.csv 2>/dev/null
for i in 0 1; do ncu -i gpurun_out/wsp.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 2>/dev/null | gzip > gpurun_out/wsp_src$i.csv.gz; done
rm -f gpurun_out/wsp.ncu-rep
tail -3 gpurun_out/wsp_ncu.log
