#!/bin/bash
# Iteration: build, selected GPU tests, one bench line, optional ncu --set full of $NCU_KERNELS
# (raw + SASS source pages as CSV).  TAG names the outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-it}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -30 gpurun_out/${T}_build.log; exit 1; }
if [[ -n "${TESTS:-}" ]]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$TESTS" > gpurun_out/${T}_tests.log 2>&1
  tail -5 gpurun_out/${T}_tests.log
fi
if [[ -z "${NO_BENCH:-}" ]]; then
timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 ${BENCH_ARGS:-} > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python - "$T" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/{t}_bench.json").read().strip().splitlines()[-1])
    print("value", d["value"], "step ms", d["ms_per_step"])
    for k, v in d["phases"].items(): print(f"  {k:9s} {v['ms']:.3f} ms")
    print("ab", json.dumps(d.get("ab")))
except Exception as e:
    print("bench failed", e); print(open(f"gpurun_out/{t}_bench.err").read()[-3000:])
PY
fi
if [[ -n "${NCU_KERNELS:-}" ]]; then
  timeout ${NCU_TIMEOUT:-900} ncu --set full --clock-control none --import-source on --profile-from-start off \
     -k regex:"${NCU_KERNELS}" -c ${NCU_COUNT:-3} -o gpurun_out/${T}_ncu -f \
     python bench.py --profile-step ${BENCH_ARGS:-} > gpurun_out/${T}_ncu.log 2>&1
  tail -3 gpurun_out/${T}_ncu.log
  ncu -i gpurun_out/${T}_ncu.ncu-rep --page raw --csv > gpurun_out/${T}_ncu_raw.csv 2>/dev/null
  for i in $(seq 0 $(( ${NCU_COUNT:-3} - 1 ))); do
    ncu -i gpurun_out/${T}_ncu.ncu-rep --page source --csv --print-source sass --launch-skip $i --launch-count 1 > gpurun_out/${T}_ncu_src$i.csv 2>/dev/null
  done
fi
