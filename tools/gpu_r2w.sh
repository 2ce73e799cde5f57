#!/bin/bash
# HVP-only G8 node sums (FEM_HVP_G8, second metadata layout): full -m gpu suite, device-timed
# A/B against FEM_HVP_G8=0, bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2w_build.log 2>&1 || { tail -20 gpurun_out/r2w_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2w_gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2w_gputests.log
for FL in "" "-DFEM_HVP_G8=0" "" "-DFEM_HVP_G8=0"; do
  FEM_NVCC_FLAGS="$FL" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/r2w_b.log 2>&1 || { echo "build failed $FL"; continue; }
  echo "[$FL] $(timeout 600 python tools/time_ops.py 2>&1 | tail -1)"
done
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
timeout 900 python bench.py --steps 10 > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2w_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "step", d["ms_per_step"], {k: round(v["ms"], 3) for k, v in d["phases"].items()})
print({k: round(v, 3) for k, v in d["ab"].items() if isinstance(v, float)})
PY
