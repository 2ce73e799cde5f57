#!/bin/bash
# Newton solve wall times (bench order: MF fixed, CSR fixed, MF inexact, CSR inexact) with the
# problem-owned Newton workspace; Newton tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r_build.log 2>&1 || { tail -20 gpurun_out/r2r_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "newton or homogen or minres" > gpurun_out/r2r_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2r_tests.log
for i in 1 2; do echo "run $i: $(timeout 900 python tools/time_newton.py 2>&1 | tail -1)"; done
timeout 900 python bench.py --steps 10 > gpurun_out/r2r_bench.json 2> gpurun_out/r2r_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2r_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "step", d["ms_per_step"], {k: round(v, 3) for k, v in d["solve"].items() if k.endswith("_s")})
PY
