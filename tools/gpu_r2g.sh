#!/bin/bash
# SoA vs odd-stride assembly records: schedule statistics, timing, ncu counters of k_rows_tile.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1 || { tail -20 gpurun_out/r2g_build.log; exit 1; }
q() { FEM_RT_SCHED_STATS=1 timeout 600 python bench.py --no-solve --no-cpu-baseline --steps 10 > gpurun_out/$1.json 2> gpurun_out/$1.err
  grep "rt plan" gpurun_out/$1.err | head -2
  python - gpurun_out/$1.json "$1" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], " ".join(f"{k}={v['ms']:.3f}" for k, v in d["phases"].items()))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
}
q soa1; FEM_RT_SOA_OFF=1 q soa0
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum
for v in 1 0; do
  if [ $v = 0 ]; then export FEM_RT_SOA_OFF=1; else unset FEM_RT_SOA_OFF; fi
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_rows_tile --launch-skip 1 -c 1 --csv --log-file gpurun_out/r2g_ncu_soa$v.csv python tools/prof_rows.py > gpurun_out/r2g_ncu_soa$v.log 2>&1
  echo "ncu soa=$v rc=$?"
done
unset FEM_RT_SOA_OFF
python - <<'PY'
import csv
for v in (1, 0):
    try:
        rows = list(csv.reader(open(f"gpurun_out/r2g_ncu_soa{v}.csv")))
        rows = [r for r in rows if len(r) > 10]
        h = rows[0]
        mi, vi = h.index("Metric Name"), h.index("Metric Value")
        print("soa", v, "; ".join(f"{r[mi]}={r[vi]}" for r in rows[1:]))
    except Exception as e:
        print("soa", v, "parse failed", e)
PY
