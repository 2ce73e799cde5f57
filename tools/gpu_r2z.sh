#!/bin/bash
# Final tree: full -m gpu suite, cfg 2 and unstructured Delaunay bench lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2z_build.log 2>&1 || { tail -20 gpurun_out/r2z_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r2z_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2z_gputests.log
timeout 900 python bench.py --config 2 --steps 20 > gpurun_out/r2z_cfg2.json 2> gpurun_out/r2z_cfg2.err; echo "cfg2 rc=$?"
timeout 1500 python bench.py --config 6 --no-solve --no-cpu-baseline --steps 10 > gpurun_out/r2z_delaunay.json 2> gpurun_out/r2z_delaunay.err; echo "delaunay rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/r2z_cfg2.json", "gpurun_out/r2z_delaunay.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], {k: round(v["ms"], 4) for k, v in d["phases"].items()})
PY
