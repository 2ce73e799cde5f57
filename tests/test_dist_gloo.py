"""Multi-rank host logic on CPU (world size 2, gloo): element partition, halo plan, halo add
in ascending rank order, owned-DOF dot products and the energy sum — checked against the
single-domain oracle.  The per-rank element work is the oracle on the rank's submesh; the
exchange uses torch.distributed with the same pack / combine rules libfem uses with NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fem_inputs as fi
from paper_2602_12365_b200 import dist as fd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mesh(kind):
    if kind == "slab":
        return None
    m = fi.roller_bc(fi.perturb(fi.grid_tet4(4, 3, 5), 0.1, 3).copy_with(material=1), 0.05)
    return m


def _worker(rank, size, port, kind, q):
    try:
        import oracle
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=size)
        if kind == "slab":
            local, gids = fd.slab_mesh(3, 2, 2, size, rank, perturb_a=0.1)
        else:
            glob = _mesh(kind)
            owner = fd.rcb_partition(glob, size)
            local, gids = fd.submesh(glob, owner, rank)
        all_ids = [None] * size
        dist.all_gather_object(all_ids, gids)
        plan = fd.halo_plan(all_ids, rank)
        o = oracle.Oracle(local)
        dim = local.dim
        # global state evaluated at this rank's nodes (generic, deterministic in global id)
        rng = np.random.default_rng(7)
        n_glob = int(max(int(a.max()) for a in all_ids)) + 1
        zg = rng.uniform(-0.003, 0.003, (n_glob, dim))
        vg = rng.uniform(-1.0, 1.0, (n_glob, dim))
        z = (zg[gids] + 0.05 * np.outer(local.coords[:, 0], np.eye(dim)[0])).ravel()
        v = vg[gids].ravel()
        z[local.dirichlet_dofs] = local.dirichlet_vals
        w = v.copy()
        w[local.dirichlet_dofs] = 0.0
        r_loc = o.residual(z)
        y_loc = o.hvp(z, w)

        def halo(y):
            yy = y.reshape(-1, dim)
            reqs, recv = [], np.zeros((len(plan.nbr_nodes), dim))
            bufs = []
            for k, qr in enumerate(plan.nbr_rank):
                seg = slice(plan.nbr_offset[k], plan.nbr_offset[k + 1])
                sb = torch.from_numpy(np.ascontiguousarray(yy[plan.nbr_nodes[seg]]))
                rb = torch.zeros(sb.shape, dtype=torch.float64)
                reqs.append(dist.isend(sb, int(qr)))
                reqs.append(dist.irecv(rb, int(qr)))
                bufs.append((seg, rb))
            for rq in reqs:
                rq.wait()
            for seg, rb in bufs:
                recv[seg] = rb.numpy()
            out = yy.copy()
            for n, lst in fd.combine_order(plan):
                s = np.zeros(dim)
                for _, t in lst:
                    s = s + (yy[n] if t < 0 else recv[t])
                out[n] = s
            return out.ravel()

        r = halo(r_loc)
        y = halo(y_loc)
        r[local.dirichlet_dofs] = 0.0
        y[local.dirichlet_dofs] = v[local.dirichlet_dofs]
        owned = np.repeat(plan.owned.astype(bool), dim)
        rr = torch.tensor([float(r[owned] @ r[owned])], dtype=torch.float64)
        dist.all_reduce(rr)
        e = torch.tensor([o.energy(z)], dtype=torch.float64)
        dist.all_reduce(e)
        q.put((rank, gids, r, y, z, v, float(rr[0]), float(e[0])))
        dist.destroy_process_group()
    except Exception as ex:  # surface worker failures to the test
        q.put(("error", repr(ex)))


@pytest.mark.parametrize("kind", ["rcb", "slab"])
def test_two_rank_halo_matches_single_domain(oracle_mod, kind):
    size = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, kind, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(size)]
    for p in procs:
        p.join(timeout=60)
    for x in res:
        assert x[0] != "error", x[1]
    res.sort(key=lambda t: t[0])
    # single-domain reference on the global mesh
    if kind == "slab":
        parts = [fd.slab_mesh(3, 2, 2, size, r, perturb_a=0.1) for r in range(size)]
        n_glob = int(max(g.max() for _, g in parts)) + 1
        coords = np.zeros((n_glob, 3))
        for m, g in parts:
            coords[g] = m.coords
        glob = fi.roller_bc(fi.grid_tet4(3, 2, 4).copy_with(coords=coords, material=1), 0.05)
    else:
        glob = _mesh(kind)
    dim = glob.dim
    zg = np.zeros((glob.n_nodes, dim))
    vg = np.zeros((glob.n_nodes, dim))
    for _, gids, r, y, z, v, *_ in res:
        zg[gids] = z.reshape(-1, dim)
        vg[gids] = v.reshape(-1, dim)
    o = oracle_mod.Oracle(glob)
    rg = o.residual(zg.ravel(), bc=True).reshape(-1, dim)
    yg = o.hvp(zg.ravel(), vg.ravel(), bc=True).reshape(-1, dim)
    for _, gids, r, y, *_ in res:
        assert np.abs(r.reshape(-1, dim) - rg[gids]).max() <= 1e-13 * np.abs(rg).max()
        assert np.abs(y.reshape(-1, dim) - yg[gids]).max() <= 1e-13 * np.abs(yg).max()
    # shared nodes carry identical bits on both ranks
    g0, g1 = res[0][1], res[1][1]
    common, i0, i1 = np.intersect1d(g0, g1, return_indices=True)
    assert len(common) > 0
    for k in (2, 3):  # r, y
        a = res[0][k].reshape(-1, dim)[i0]
        b = res[1][k].reshape(-1, dim)[i1]
        assert np.array_equal(a, b)
    # owned-DOF dot and energy sum equal the global ones
    assert abs(res[0][6] - float(rg.ravel() @ rg.ravel())) <= 1e-12 * float(rg.ravel() @ rg.ravel())
    assert res[0][6] == res[1][6]
    eg = o.energy(zg.ravel())
    assert abs(res[0][7] - eg) <= 1e-13 * abs(eg)


def test_partitions_cover_elements_once():
    m = _mesh("rcb")
    for parts in (2, 3, 4):
        owner = fd.rcb_partition(m, parts)
        assert set(np.unique(owner)) == set(range(parts))
        counts = np.bincount(owner)
        assert counts.max() - counts.min() <= 1
        ids = [fd.submesh(m, owner, r)[1] for r in range(parts)]
        plans = [fd.halo_plan(ids, r) for r in range(parts)]
        # every node owned by exactly one rank
        own = np.zeros(m.n_nodes, int)
        for pl in plans:
            own[pl.global_ids[pl.owned.astype(bool)]] += 1
        assert np.all(own == 1)
        # neighbour relation symmetric with equal shared-node lists
        for pl in plans:
            for k, q in enumerate(pl.nbr_rank):
                other = plans[q]
                kk = list(other.nbr_rank).index(pl.rank)
                a = pl.global_ids[pl.nbr_nodes[pl.nbr_offset[k]:pl.nbr_offset[k + 1]]]
                b = other.global_ids[other.nbr_nodes[other.nbr_offset[kk]:other.nbr_offset[kk + 1]]]
                assert np.array_equal(a, b)
