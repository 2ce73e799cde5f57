"""The real NCCL exchange under torchrun, two ranks on two GPUs:
fem_residual / fem_hvp with the overlapped interface-first halo add, fem_spmv on the local
CSRs, fem_energy and fem_cg_solve with allreduced owned-DOF dots — against the single-domain
oracle (tests/_nccl_worker.py).  NCCL refuses two ranks on one device, so this skips on
boxes with fewer than two GPUs (the one-GPU emulation is tests/test_gpu_dist.py)."""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_torchrun_nccl_halo_cg(world):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (NCCL allows one rank per device)")
    from paper_2602_12365_b200 import build
    build.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(_port()), os.path.join(ROOT, "tests", "_nccl_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert r.stdout.count("rank ") == world
