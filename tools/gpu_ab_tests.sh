#!/bin/bash
# Default build + a GPU test selection ($TESTS), then compile-flag A/B variants (args).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/abt_build.log 2>&1 || { tail -30 gpurun_out/abt_build.log; exit 1; }
if [[ -n "${TESTS:-}" ]]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$TESTS" > gpurun_out/abt_tests.log 2>&1
  tail -4 gpurun_out/abt_tests.log
fi
bash tools/ab_flags.sh "" "$@"
