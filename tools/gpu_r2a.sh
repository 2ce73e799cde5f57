#!/bin/bash
# Round-2 coverage run: environment, full -m gpu suite (incl. cfg4 / Delaunay-3D / NCCL tests),
# cfg4 strong-mode P=1 bench line, default bench line.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-r2a}
{ free -g; nvidia-smi -L; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"; } > gpurun_out/${T}_env.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail -20 gpurun_out/${T}_build.log; exit 1; }
timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/${T}_tests.log 2>&1
tail -30 gpurun_out/${T}_tests.log
if [[ -z "${NO_BENCH:-}" ]]; then
timeout 900 python bench.py --scaling strong --no-solve --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/${T}_strong.json 2> gpurun_out/${T}_strong.err
tail -c 600 gpurun_out/${T}_strong.json; tail -5 gpurun_out/${T}_strong.err
timeout 900 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -c 600 gpurun_out/${T}_bench.json; tail -5 gpurun_out/${T}_bench.err
fi
