#!/bin/bash
# Stream-ordered pool allocations in the pattern / coloring setup: full -m gpu suite, then two
# bench lines (setup medians of fresh problems).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2n_build.log 2>&1 || { tail -20 gpurun_out/r2n_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2n_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2n_tests.log
for i in 1 2; do
  timeout 900 python bench.py --no-solve --no-cpu-baseline --steps 10 > gpurun_out/r2n_bench$i.json 2> gpurun_out/r2n_bench$i.err
  python - gpurun_out/r2n_bench$i.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
s = d["setup"]
print("pattern", [round(x, 1) for x in s["pattern_ms_samples"]], "first", round(s["pattern_ms_first"], 1),
      "| coloring", [round(x, 1) for x in s["coloring_ms_samples"]], "first", round(s["coloring_ms_first"], 1),
      "| assembly", round(d["assembly_ms"], 3))
PY
done
