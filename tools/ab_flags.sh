#!/bin/bash
# A/B over compile-time variants: each argument is a set of nvcc -D flags; one quick bench
# line per variant (assembly / HVP / residual ms printed), then the default build restored.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
i=0
for FL in "$@"; do
  i=$((i+1))
  FEM_NVCC_FLAGS="$FL" python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > gpurun_out/ab_build$i.log 2>&1 || { echo "build failed: $FL"; tail -5 gpurun_out/ab_build$i.log; continue; }
  timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 ${BENCH_ARGS:-} > gpurun_out/ab$i.json 2> gpurun_out/ab$i.err
  python - "$FL" gpurun_out/ab$i.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    ph = d["phases"]
    print(f"[{sys.argv[1]}] " + " ".join(f"{k}={v['ms']:.3f}" for k, v in ph.items()))
except Exception as e:
    print(f"[{sys.argv[1]}] failed: {e}")
PY
done
python -c "from paper_2602_12365_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
