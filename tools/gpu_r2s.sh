#!/bin/bash
# Push-form greedy coloring (FEM_COLOR_PUSH): bit-exact coloring tests, setup timing A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2s_build.log 2>&1 || { tail -20 gpurun_out/r2s_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -k "color or assembly or smoke or delaunay or cfg4" > gpurun_out/r2s_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2s_tests.log
q() { timeout 900 python bench.py --no-solve --no-cpu-baseline --steps 5 > gpurun_out/$1.json 2> gpurun_out/$1.err
  python - gpurun_out/$1.json $1 <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
s = d["setup"]
print(sys.argv[2], "coloring", [round(x, 1) for x in s["coloring_ms_samples"]], "first", round(s["coloring_ms_first"], 1), "colors", s["n_colors"], "pattern", round(s["pattern_ms"], 1))
PY
}
q push1
FEM_NVCC_FLAGS="-DFEM_COLOR_PUSH=0" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1 && q push0
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
