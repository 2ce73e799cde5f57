#!/bin/bash
# bench.py under torchrun with one rank (the driver's launch form for N > 1), weak and strong.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2aa_build.log 2>&1 || { tail -20 gpurun_out/r2aa_build.log; exit 1; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/r2aa_weak.json 2> gpurun_out/r2aa_weak.err; echo "weak rc=$?"; tail -c 400 gpurun_out/r2aa_weak.json; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --scaling strong --steps 3 --warmup 3 --no-solve --no-cpu-baseline > gpurun_out/r2aa_strong.json 2> gpurun_out/r2aa_strong.err; echo "strong rc=$?"; tail -c 400 gpurun_out/r2aa_strong.json; echo
