"""bench.py's multi-GPU workload accounting on CPU.

* DOF / element counts of the weak and strong scaling plans (closed forms).
* The strong plan's z-slabs (BASELINE cfg 4: 256 z-cells cut into P slabs of 256/P) cover
  every element of the global block exactly once, and their nodes cover every global node,
  for P = 2, 4, 8 — checked by world-size-P gloo process groups that gather every rank's
  elements as global node tuples.  The x/y extent is reduced (the z split under test does
  not depend on it; a 255 x 255 slab per process would be ~10^8 elements).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import fem_inputs as fi  # noqa: E402
from paper_2602_12365_b200 import dist as fd  # noqa: E402


def test_strong_plan_is_cfg4_for_every_p():
    for P in (1, 2, 4, 8):
        p = bench.scaling_plan("strong", P)
        assert (p["nx"], p["ny"], p["nz_total"]) == (255, 255, 256)
        assert p["nz_per_rank"] * P == 256
        assert p["n_global_dofs"] == 50_528_256          # BASELINE cfg 4 / SURVEY §8 table
        assert p["n_global_elems"] == 99_878_400
    with pytest.raises(SystemExit):
        bench.scaling_plan("strong", 3)                   # 256 cells do not split into 3


def test_weak_plan_is_cfg3_per_gpu():
    p1 = bench.scaling_plan("weak", 1)
    assert p1["n_global_dofs"] == 10_328_853 and p1["n_global_elems"] == 20_250_000
    for P in (2, 4, 8):
        p = bench.scaling_plan("weak", P)
        assert p["n_global_dofs"] == 3 * 151 * 151 * (150 * P + 1)
        assert p["n_global_elems"] == P * 20_250_000


def test_single_slab_is_the_cfg4_mesh():
    """P = 1 of the strong plan is fi.config_mesh(4): same coordinates (perturbation drawn per
    global node with the same seed) and the same Dirichlet set."""
    n = 6
    p = bench.scaling_plan("strong", 1, n=n)
    m, gids = fd.slab_mesh(p["nx"], p["ny"], p["nz_per_rank"], 1, 0, perturb_a=0.1, seed=p["seed"])
    g = fi.roller_bc(fi.perturb(fi.grid_tet4(n, n, n + 1), 0.1, seed=14).copy_with(material=1), 0.05)
    assert np.array_equal(gids, np.arange(g.n_nodes))
    assert np.array_equal(m.conn, g.conn)
    assert np.array_equal(m.coords, g.coords)
    assert np.array_equal(m.dirichlet_dofs, g.dirichlet_dofs)
    assert np.array_equal(m.dirichlet_vals, g.dirichlet_vals)
    full = fi.config_mesh(4, n=n)
    assert np.array_equal(full.coords, g.coords) and np.array_equal(full.conn, g.conn)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cover_worker(rank, size, port, nxy, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=size)
        p = bench.scaling_plan("strong", size)
        m, gids = fd.slab_mesh(nxy, nxy, p["nz_per_rank"], size, rank, perturb_a=0.1, seed=p["seed"])
        elems = np.sort(gids[m.conn], axis=1)           # elements as sorted global node tuples
        got = [None] * size
        dist.all_gather_object(got, (elems, gids, m.n_total))
        if rank == 0:
            glob = fi.grid_tet4(nxy, nxy, p["nz_total"])
            want = np.sort(glob.conn.astype(np.int64), axis=1)
            allv = np.concatenate([e for e, _, _ in got])
            assert len(allv) == len(want) == 6 * nxy * nxy * 256
            a = np.unique(allv, axis=0, return_counts=True)
            assert (a[1] == 1).all(), "an element is on two ranks"
            assert np.array_equal(a[0], np.unique(want, axis=0)), "element sets differ"
            nodes = np.unique(np.concatenate([g for _, g, _ in got]))
            assert np.array_equal(nodes, np.arange(glob.n_nodes))
            # interface planes: every slab boundary shares (nxy+1)^2 nodes with its neighbour
            shared = sum(d for _, _, d in got) // 3 - glob.n_nodes
            assert shared == (size - 1) * (nxy + 1) ** 2
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, None))
    except Exception as ex:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("P", [2, 4, 8])
def test_strong_slabs_cover_cfg4_exactly_once(P):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cover_worker, args=(r, P, port, 3, q)) for r in range(P)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(P)]
    for pr in procs:
        pr.join(timeout=60)
    errs = [e for _, e in res if e]
    assert not errs, errs[0]
