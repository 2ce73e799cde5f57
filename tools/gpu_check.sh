#!/bin/bash
# Iteration check in one call: build, -m gpu suite (PYTEST_K narrows it), quick bench (no
# solves / CPU baseline) with its phases and A/B entries printed.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-chk}
if [ -n "${FEM_NVCC_FLAGS:-}" ]; then  # compile-time variant: force the rebuild
  python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
fi
python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${T}_gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/${T}_gputests.log
  tail -4 gpurun_out/${T}_gputests.log
fi
timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 ${BENCH_ARGS:-} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python - gpurun_out/${T}_bench.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print("value", round(d["value"], 3), "step", round(d["ms_per_step"], 3))
    print(" ".join(f"{k}={v['ms']:.3f}" for k, v in d["phases"].items()))
    print(" ".join(f"{k}={v:.3f}" for k, v in d["ab"].items() if isinstance(v, float)))
except Exception as e:
    print("bench failed", e); print(open(sys.argv[1].replace('.json','.err')).read()[-2000:])
PY
