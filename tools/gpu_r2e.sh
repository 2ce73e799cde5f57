#!/bin/bash
# Session check after the checkpoint restore: build, the -m gpu suite, a quick bench line,
# and the DOF sweep on the round-2 kernels (profiles/r02_sweep*).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=r2e bash tools/gpu_check.sh
timeout 1500 python tools/sweep.py gpurun_out/r02 > gpurun_out/r02_sweep.log 2>&1; echo "sweep rc=$?"
tail -5 gpurun_out/r02_sweep.log
