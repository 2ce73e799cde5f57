#!/bin/bash
# Colored Alg. 2 node tiles: CTA size (FEM_CT_THREADS) and seeds per tile (FEM_CT_NT) A/B, with
# the colored-assembly parity tests on the default.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2o_build.log 2>&1 || { tail -20 gpurun_out/r2o_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -k "colored or assembly or full_size or delaunay or cfg4" > gpurun_out/r2o_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2o_tests.log
BENCH_ARGS="" bash tools/ab_flags.sh "" "-DFEM_CT_THREADS=256 -DFEM_CT_MINB=2" "-DFEM_CT_THREADS=128 -DFEM_CT_MINB=4 -DFEM_CT_NT=8" "-DFEM_CT_THREADS=128 -DFEM_CT_MINB=4" "-DFEM_CT_THREADS=64 -DFEM_CT_NT=2" "-DFEM_CT_THREADS=32 -DFEM_CT_MINB=16 -DFEM_CT_NT=2" 2>&1
for i in 1 2 3 4 5 6; do python - gpurun_out/ab$i.json $i <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], "colored", round(d["colored_assembly_ms"], 3), "rows", round(d["assembly_ms"], 3))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
