#!/bin/bash
# compute-sanitizer memcheck + racecheck over the small-mesh GPU parity tests: every kernel
# of the library on cfg1, the 3D NH mesh and the 3D Delaunay mesh (all residual / HVP modes incl.
# the TMA-bulk streamed geometry, colored passes, linearized HVP; all assembly modes), the MPC
# mesh, the virtual-work and solver tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
T=${TAG:-san}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1
SEL='cfg1-2d-le or 3d-nh] or 3d-nh-delaunay or 2d-le-mpc or vw or minres or loads or linearized or 32_lanes'
timeout 2400 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 7 \
  python -m pytest tests/test_gpu_parity.py tests/test_gpu_vw.py tests/test_gpu_homogenization.py tests/test_gpu_loads.py \
  -m gpu -q -x -p no:cacheprovider -k "$SEL" > gpurun_out/${T}_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -3 gpurun_out/${T}_memcheck.log
timeout 2400 compute-sanitizer --tool racecheck --error-exitcode 7 \
  python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
  -k "(cfg1-2d-le or 3d-nh] or 3d-nh-delaunay) and (test_residual or test_hvp or modes or assembly or linearized)" > gpurun_out/${T}_racecheck.log 2>&1
echo "racecheck rc=$?"; tail -3 gpurun_out/${T}_racecheck.log
