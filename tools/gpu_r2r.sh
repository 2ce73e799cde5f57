#!/bin/bash
# Newton solve wall times with the Newton work buffer from the stream-ordered pool; Newton tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2r_build.log 2>&1 || { tail -20 gpurun_out/r2r_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "newton or homogen or minres" > gpurun_out/r2r_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2r_tests.log
for i in 1 2 3; do echo "run $i: $(timeout 900 python tools/time_newton.py 2>&1 | tail -1)"; done
