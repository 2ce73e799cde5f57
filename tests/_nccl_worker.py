"""torchrun worker for tests/test_gpu_nccl.py: one rank per GPU, the real NCCL halo path.

Each rank holds an RCB element partition of a 3D NH mesh, creates its problem with a halo plan
and an NCCL communicator (overlapped interface-first residual / HVP), and checks its owned and
shared DOFs of fem_residual, fem_hvp, fem_spmv (local CSR + halo add), fem_energy (allreduce)
and fem_cg_solve (owned-DOF dots + allreduce) against the single-domain CPU oracle; shared
DOFs must carry identical bits on every rank (ascending-rank summation)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import fem_inputs as fi  # noqa: E402
import oracle  # noqa: E402
from paper_2602_12365_b200 import dist as fd  # noqa: E402
from paper_2602_12365_b200 import fem  # noqa: E402

TOL = 1e-12


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    glob = fi.roller_bc(fi.perturb(fi.grid_tet4(9, 8, 10), 0.1, 4).copy_with(material=1), 0.05)
    owner = fd.rcb_partition(glob, world)
    mesh, gids = fd.submesh(glob, owner, rank)
    ids = [None] * world
    dist.all_gather_object(ids, gids)
    plan = fd.halo_plan(ids, rank)
    uid = [fem.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = fem.nccl_comm_init(uid[0], rank, world)
    assert fem.nccl_comm_count(comm) == world
    prob = fem.Problem(mesh, plan=plan, nccl_comm=comm)
    d = 3
    z = fi.lift(glob, fi.generic_state(glob, 3))
    v = fi.random_direction(glob.n_total, 4)
    zl = torch.as_tensor(z.reshape(-1, d)[gids].ravel(), device="cuda")
    vl = torch.as_tensor(v.reshape(-1, d)[gids].ravel(), device="cuda")
    ro = oracle.Oracle(glob)
    sel = (gids[:, None] * d + np.arange(d)).ravel()
    checks = {}
    for bc in (False, True):
        rr = ro.residual(z, bc=bc)
        yr = ro.hvp(z, v, bc=bc)
        r = prob.residual(zl, bc=bc).cpu().numpy()
        y = prob.hvp(zl, vl, bc=bc).cpu().numpy()
        checks[f"residual bc={bc}"] = np.abs(r - rr[sel]).max() / np.abs(rr).max()
        checks[f"hvp bc={bc}"] = np.abs(y - yr[sel]).max() / np.abs(yr).max()
    e = prob.energy(zl).item()
    er = ro.energy(z)
    checks["energy"] = abs(e - er) / abs(er)
    vals = prob.assemble_csr(zl, bc=True)                 # local CSR (unassembled interface)
    ys = prob.spmv(vals, vl).cpu().numpy()
    yr = ro.hvp(z, v, bc=True)
    checks["spmv"] = np.abs(ys - yr[sel]).max() / np.abs(yr).max()
    b = v.copy()
    b[glob.dirichlet_dofs] = 0.0
    xr, rinfo = ro.cg(b, op=0, z=z, rtol=1e-13)
    bl = torch.as_tensor(b.reshape(-1, d)[gids].ravel(), device="cuda")
    for op, jac in ((0, 0), (1, 1)):
        x, info = prob.cg_solve(bl, z=zl, vals=vals, op=op, rtol=1e-13, jacobi=jac)
        assert info["converged"], info
        checks[f"cg op={op}"] = np.abs(x.cpu().numpy() - xr[sel]).max() / np.abs(xr).max()
    # identical bits on shared DOFs: gather every rank's HVP and compare on common nodes
    y = prob.hvp(zl, vl, bc=True).cpu().numpy().reshape(-1, d)
    allys = [None] * world
    dist.all_gather_object(allys, y)
    for q in range(world):
        if q != rank:
            common, ia, ib = np.intersect1d(gids, ids[q], return_indices=True)
            assert len(common) > 0 or q not in plan.nbr_rank
            assert np.array_equal(y[ia], allys[q][ib]), f"shared DOFs differ with rank {q}"
    bad = {k: x for k, x in checks.items() if not x <= (1e-10 if k.startswith("cg") else TOL)}
    print(f"rank {rank}: " + " ".join(f"{k}={x:.2e}" for k, x in checks.items()), flush=True)
    del prob
    torch.cuda.synchronize()
    fem.nccl_comm_destroy(comm)
    dist.destroy_process_group()
    if bad:
        raise SystemExit(f"rank {rank} parity failures: {bad}")


if __name__ == "__main__":
    main()
