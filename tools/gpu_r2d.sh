#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-r2d}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -30 gpurun_out/${T}_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1
tail -6 gpurun_out/${T}_tests.log
timeout 600 python tools/timeline.py --tag ${T} > gpurun_out/${T}_timeline.log 2>&1; tail -30 gpurun_out/${T}_timeline.log
cp profiles/${T}_cg_timeline* gpurun_out/ 2>/dev/null
timeout 900 python bench.py --config 2 --steps 20 > gpurun_out/${T}_cfg2.json 2> gpurun_out/${T}_cfg2.err
tail -c 300 gpurun_out/${T}_cfg2.json; tail -3 gpurun_out/${T}_cfg2.err
