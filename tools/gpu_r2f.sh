#!/bin/bash
# SoA assembly records (FEM_RT_SOA; FEM_RT_SOA_OFF=1 = odd-stride records) and the log
# constant table (FEM_LOG_CTAB) A/Bs on the quick bench, the parity tests they touch
# (assembly, Newton incl. Eisenstat-Walker forcing), then one full bench line with solves.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2f_build.log 2>&1 || { tail -20 gpurun_out/r2f_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q -k "assembly or rows or row_ or newton or energy or hvp or residual or full_size or cfg4 or delaunay" > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r2f_tests.log
q() { timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 > gpurun_out/$1.json 2> gpurun_out/$1.err
  python - gpurun_out/$1.json "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], " ".join(f"{k}={v['ms']:.3f}" for k, v in d["phases"].items()), "colored", round(d["colored_assembly_ms"], 3))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
}
q soa1; FEM_RT_SOA_OFF=1 q soa0; q soa1b; FEM_RT_SOA_OFF=1 q soa0b
bash tools/ab_flags.sh "-DFEM_LOG_CTAB=0" "-DFEM_LOG_CTAB=1"
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2f_bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "step", d["ms_per_step"], "assembly", d["assembly_ms"])
s = d.get("solve", {})
for k in ("newton_s", "newton_csr_s", "newton_ew_s", "newton_csr_ew_s"):
    print(k, s.get(k), s.get(k[:-2]))
print("ew vs fixed", s.get("newton_ew_vs_fixed_maxdiff"), s.get("newton_csr_ew_vs_fixed_maxdiff"))
PY
