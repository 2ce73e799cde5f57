#!/bin/bash
# Final tree (component-wise node staging): full -m gpu suite, smoke, bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2ac_build.log 2>&1 || { tail -20 gpurun_out/r2ac_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2ac_gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2ac_gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ac_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2ac_bench.json 2> gpurun_out/r2ac_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2ac_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "step", d["ms_per_step"], {k: round(v["ms"], 3) for k, v in d["phases"].items()})
print("lin", round(d["ab"]["hvp_linearized_ms"], 3), {k: round(v, 3) for k, v in d["solve"].items() if k.endswith("_s")})
PY
