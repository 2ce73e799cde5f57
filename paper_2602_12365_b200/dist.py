"""Element partition and halo plan for multi-GPU runs — host-side setup.

The global functional is a sum of element contributions, so the mesh is
split by elements: z-slabs for the structured configs, recursive coordinate bisection (RCB)
of element centroids in general.  Each rank keeps the nodes its elements touch, numbered
in ascending global id.  Nodes shared between ranks form the interface; each residual / HVP
/ SpMV needs one halo add over them, in which every rank sums the partials of a shared DOF
in ascending rank order (so all ranks hold the same bits).  A node is owned by the lowest
rank touching it; dot products run over owned DOFs.

This module only builds index arrays (numpy); the exchange itself runs inside libfem
(NCCL) or, for tests, through `emulate_halo_add` / torch.distributed.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

import fem_inputs as fi


@dataclass
class HaloPlan:
    rank: int
    size: int
    global_ids: np.ndarray      # [n_local_nodes] int64, ascending
    nbr_rank: np.ndarray        # [n_nbr] int32, ascending
    nbr_offset: np.ndarray      # [n_nbr+1] int64
    nbr_nodes: np.ndarray       # [nbr_offset[-1]] int32 local node ids, ascending global id per nbr
    owned: np.ndarray           # [n_local_nodes] uint8


def rcb_partition(mesh: fi.Mesh, parts: int) -> np.ndarray:
    """Element -> rank by recursive coordinate bisection of centroids (deterministic)."""
    cent = mesh.coords[mesh.conn].mean(axis=1)
    owner = np.zeros(mesh.n_elems, np.int32)

    def split(idx, lo, n):
        if n == 1 or len(idx) == 0:
            owner[idx] = lo
            return
        axis = int(np.argmax(np.ptp(cent[idx], axis=0)))
        order = idx[np.argsort(cent[idx, axis], kind="stable")]
        n_left = n // 2
        cut = len(order) * n_left // n
        split(order[:cut], lo, n_left)
        split(order[cut:], lo + n_left, n - n_left)

    split(np.arange(mesh.n_elems), 0, parts)
    return owner


def submesh(mesh: fi.Mesh, elem_owner: np.ndarray, rank: int):
    """Rank-local mesh (nodes in ascending global id) and its global node ids."""
    elems = np.nonzero(elem_owner == rank)[0]
    gconn = mesh.conn[elems]
    gids = np.unique(gconn)
    lconn = np.searchsorted(gids, gconn).astype(np.int32)
    m = mesh.dim
    keep = {}
    if len(mesh.dirichlet_dofs):
        gnode = mesh.dirichlet_dofs // m
        pos = np.searchsorted(gids, gnode)
        ok = (pos < len(gids)) & (gids[np.minimum(pos, len(gids) - 1)] == gnode)
        keep["dirichlet_dofs"] = (pos[ok] * m + mesh.dirichlet_dofs[ok] % m).astype(np.int32)
        keep["dirichlet_vals"] = mesh.dirichlet_vals[ok]
    if mesh.n_mpc:
        raise ValueError("multi-point constraints with more than one rank are out of scope")
    local = mesh.copy_with(coords=mesh.coords[gids], conn=lconn,
                           phase=None if mesh.phase is None else mesh.phase[elems],
                           f_ext=None if mesh.f_ext is None else
                           mesh.f_ext.reshape(-1, m)[gids].ravel(), **keep)
    return local, gids.astype(np.int64)


def slab_mesh(nx: int, ny: int, nz_per_rank: int, size: int, rank: int, material=fi.NEO_HOOKEAN,
              eps: float = 0.05, perturb_a: float = 0.0, seed: int = 13):
    """Rank `rank`'s z-slab of an nx x ny x (nz_per_rank*size) Kuhn block (weak scaling),
    with the roller stretch of the global block.  Returns (local mesh, global node ids)."""
    nz_total = nz_per_rank * size
    z0 = nz_per_rank * rank
    m = fi.grid_tet4(nx, ny, nz_per_rank, z0=z0, nz_total=nz_total)
    m = m.copy_with(material=material, shape=(nx, ny, nz_total))
    gids = np.arange(m.n_nodes, dtype=np.int64) + z0 * (nx + 1) * (ny + 1)
    if perturb_a:
        # jitter from a global stream so partitions agree on shared nodes
        rng = np.random.default_rng(seed)
        h = 1.0 / max(nx, ny, nz_total)
        n_glob = (nx + 1) * (ny + 1) * (nz_total + 1)
        jit = rng.uniform(-perturb_a * h, perturb_a * h, size=(n_glob, 3))[gids]
        interior = ~fi.boundary_node_mask(m, length=1.0)
        coords = m.coords.copy()
        coords[interior] += jit[interior]
        m = m.copy_with(coords=coords)
    m = fi.roller_bc(m, eps)
    # roller_bc marks planes of the LOCAL slab; keep only the global boundary planes
    dofs, vals = m.dirichlet_dofs, m.dirichlet_vals
    node, comp = dofs // 3, dofs % 3
    z = m.coords[node, 2]
    keep = ~((comp == 2) & (np.abs(z) > 1e-12))          # u_z = 0 only on the global z = 0
    return m.copy_with(dirichlet_dofs=dofs[keep], dirichlet_vals=vals[keep]), gids


def halo_plan(all_global_ids: list, rank: int) -> HaloPlan:
    """Neighbour lists and ownership from every rank's sorted global node ids."""
    size = len(all_global_ids)
    mine = all_global_ids[rank]
    nbr_rank, offs, nodes = [], [0], []
    owned = np.ones(len(mine), np.uint8)
    for q in range(size):
        if q == rank:
            continue
        common, li, _ = np.intersect1d(mine, all_global_ids[q], assume_unique=True,
                                       return_indices=True)
        if len(common) == 0:
            continue
        nbr_rank.append(q)
        nodes.append(li.astype(np.int32))          # ascending global id
        offs.append(offs[-1] + len(li))
        if q < rank:
            owned[li] = 0
    return HaloPlan(rank, size, mine, np.asarray(nbr_rank, np.int32), np.asarray(offs, np.int64),
                    np.concatenate(nodes) if nodes else np.zeros(0, np.int32), owned)


def combine_order(plan: HaloPlan):
    """For every shared local node: its contributions in ascending rank order, as
    (node, [(rank, position-in-recv-buffer or -1 for self), ...])."""
    contrib = {}
    for k, q in enumerate(plan.nbr_rank):
        for t in range(plan.nbr_offset[k], plan.nbr_offset[k + 1]):
            contrib.setdefault(int(plan.nbr_nodes[t]), []).append((int(q), int(t)))
    out = []
    for n in sorted(contrib):
        lst = contrib[n] + [(plan.rank, -1)]
        lst.sort()
        out.append((n, lst))
    return out


def emulate_halo_add(partials: list, plans: list, dim: int) -> list:
    """Reference halo add for P partitions held in one process (numpy): pack, exchange,
    combine in ascending rank order.  Used by tests against single-domain results."""
    send = []
    for y, pl in zip(partials, plans):
        yy = y.reshape(-1, dim)
        send.append({int(q): yy[pl.nbr_nodes[pl.nbr_offset[k]:pl.nbr_offset[k + 1]]].copy()
                     for k, q in enumerate(pl.nbr_rank)})
    out = []
    for y, pl in zip(partials, plans):
        yy = y.reshape(-1, dim).copy()
        recv = np.zeros((len(pl.nbr_nodes), dim))
        for k, q in enumerate(pl.nbr_rank):
            recv[pl.nbr_offset[k]:pl.nbr_offset[k + 1]] = send[int(q)][pl.rank]
        own = y.reshape(-1, dim)
        for n, lst in combine_order(pl):
            s = np.zeros(dim)
            for _, t in lst:
                s = s + (own[n] if t < 0 else recv[t])
            yy[n] = s
        out.append(yy.ravel())
    return out
