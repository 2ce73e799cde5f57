#!/bin/bash
# Run-time SoA assembly records against the oracle (test_row_tiles_soa_records) + row tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2u_build.log 2>&1 || { tail -20 gpurun_out/r2u_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "soa or row_tiles or rows_mode" > gpurun_out/r2u_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2u_tests.log
