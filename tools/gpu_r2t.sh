#!/bin/bash
# End-of-session check on the final tree: full -m gpu suite, smoke, bench line (with solves),
# reference arm.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2t_build.log 2>&1 || { tail -20 gpurun_out/r2t_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2t_gputests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2t_gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2t_bench.json 2> gpurun_out/r2t_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2t_bench_ref.json 2> gpurun_out/r2t_bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2t_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "step", d["ms_per_step"], "assembly", d["assembly_ms"], "setup", d["setup"]["pattern_ms"], d["setup"]["coloring_ms"])
print({k: round(v, 3) for k, v in d["solve"].items() if k.endswith("_s")})
PY
