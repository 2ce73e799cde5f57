"""Multi-rank halo add of libfem on ONE GPU: P partitions held in one process, element partial
sums with FEM_LOCAL_ONLY, fem_halo_pack -> (exchange emulated by device copies, standing in for
NCCL send/recv) -> fem_halo_combine; checked against the single-domain GPU result and the
oracle.  Shared DOFs must carry identical bits on all ranks (ascending-rank summation)."""
import numpy as np
import pytest

import fem_inputs as fi
from paper_2602_12365_b200 import dist as fd

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fem():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_12365_b200 import build, fem as f
    build.build()
    return f


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


def exchange(probs, plans, sends):
    recvs = []
    for r, pl in enumerate(plans):
        recv = torch.zeros(max(probs[r].halo_size(), 1), dtype=torch.float64, device="cuda")
        d = probs[r].dim
        for k, q in enumerate(pl.nbr_rank):
            other = plans[q]
            kk = list(other.nbr_rank).index(r)
            a, b = pl.nbr_offset[k] * d, pl.nbr_offset[k + 1] * d
            c, e = other.nbr_offset[kk] * d, other.nbr_offset[kk + 1] * d
            recv[a:b] = sends[q][c:e]
        recvs.append(recv)
    return recvs


@pytest.mark.parametrize("parts,kind", [(2, "rcb"), (3, "rcb"), (4, "slab")])
def test_local_partials_plus_halo_equal_single_domain(fem, oracle_mod, parts, kind):
    if kind == "slab":
        pieces = [fd.slab_mesh(5, 4, 2, parts, r, perturb_a=0.1) for r in range(parts)]
        n_glob = int(max(g.max() for _, g in pieces)) + 1
        coords = np.zeros((n_glob, 3))
        for m, g in pieces:
            coords[g] = m.coords
        glob = fi.roller_bc(fi.grid_tet4(5, 4, 2 * parts).copy_with(coords=coords, material=1), 0.05)
    else:
        glob = fi.roller_bc(fi.perturb(fi.grid_tet4(6, 5, 7), 0.1, 4).copy_with(material=1), 0.05)
        owner = fd.rcb_partition(glob, parts)
        pieces = [fd.submesh(glob, owner, r) for r in range(parts)]
    ids = [g for _, g in pieces]
    plans = [fd.halo_plan(ids, r) for r in range(parts)]
    probs = [fem.Problem(m, plan=pl) for (m, _), pl in zip(pieces, plans)]
    dim = 3
    z = fi.lift(glob, fi.generic_state(glob, 3))
    v = fi.random_direction(glob.n_total, 4)
    zg, vg = z.reshape(-1, dim), v.reshape(-1, dim)
    single = fem.Problem(glob)
    rs = single.residual(dev(z), bc=True).cpu().numpy().reshape(-1, dim)
    ys = single.hvp(dev(z), dev(v), bc=True).cpu().numpy().reshape(-1, dim)
    ro = oracle_mod.Oracle(glob)
    rref = ro.residual(z, bc=True).reshape(-1, dim)
    yref = ro.hvp(z, v, bc=True).reshape(-1, dim)
    for op in ("residual", "hvp"):
        locs = []
        for (m, g), pr in zip(pieces, probs):
            zl, vl = dev(zg[g].ravel()), dev(vg[g].ravel())
            if op == "residual":
                locs.append(pr.residual(zl, bc=True, flags=fem.LOCAL_ONLY))
            else:
                locs.append(pr.hvp(zl, vl, bc=True, flags=fem.LOCAL_ONLY))
        sends = [pr.halo_pack(y) for pr, y in zip(probs, locs)]
        recvs = exchange(probs, plans, sends)
        outs = [pr.halo_combine(y, rc).cpu().numpy().reshape(-1, dim)
                for pr, y, rc in zip(probs, locs, recvs)]
        ref, gpu1 = (rref, rs) if op == "residual" else (yref, ys)
        scale = np.abs(ref).max()
        for (m, g), out in zip(pieces, outs):
            assert np.abs(out - ref[g]).max() <= 1e-12 * scale
            assert np.abs(out - gpu1[g]).max() <= 1e-12 * scale
        for a in range(parts):
            for b in range(a + 1, parts):
                common, ia, ib = np.intersect1d(ids[a], ids[b], return_indices=True)
                assert np.array_equal(outs[a][ia], outs[b][ib])
    # without a communicator the collective calls must refuse, not silently skip
    with pytest.raises(fem.FemError):
        probs[0].residual(dev(zg[ids[0]].ravel()))
    with pytest.raises(fem.FemError):
        probs[0].energy(dev(zg[ids[0]].ravel()))
