#!/bin/bash
# Iteration check: build, a pytest selection (-m gpu -k "$TESTS"), one quick bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [[ -n "${TESTS:-}" ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$TESTS" > gpurun_out/iter_tests.log 2>&1
  tail -15 gpurun_out/iter_tests.log
fi
timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 ${BENCH_ARGS:-} > gpurun_out/iter_bench.json 2> gpurun_out/iter_bench.err
python - <<'PY'
import json
try:
    d = json.loads(open("gpurun_out/iter_bench.json").read().strip().splitlines()[-1])
    print("value", d["value"], "step ms", d["ms_per_step"])
    for k, v in d["phases"].items(): print(f"  {k:9s} {v['ms']:.3f} ms")
    print("ab", d.get("ab"))
except Exception as e:
    print("bench failed", e); print(open("gpurun_out/iter_bench.err").read()[-3000:])
PY
