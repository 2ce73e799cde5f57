"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module is the ONLY code both sides of a parity test share.  It
generates data — meshes, constraint sets, states — and holds none of the method's
arithmetic: no shape-function gradients, no Jacobians, no energy densities, no
derivatives.  Everything here is plain index / coordinate bookkeeping.

Conventions:
  * C5  Tri3: quad cell split along the lower-left -> upper-right diagonal, CCW:
        (a,b,c),(a,c,d); nodes row-major with x fastest; cells row-major.
        (PAPER.md is silent on meshes.)
  * C6  Tet4: Kuhn/Freudenthal split, 6 tets per cell along the axis permutations
        (0,1,2),(0,2,1),(1,0,2),(1,2,0),(2,0,1),(2,1,0); tets of odd permutations
        have their last two nodes swapped so every tet is positively oriented.
  * C7  DOF = node*m + comp (PAPER.md P:282 `u_flat.reshape(-1, n_dofs)`,
        Alg. 1 P:120 "Reshape to nodal representation"); multipliers after all u.
  * C13 periodic pairs; C15 roller / clamped stretch; C16 perturbed meshes.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

# C3: E = 1, nu = 0.3 (PAPER.md P:558 uses these values; §5 does not state any)
E_DEFAULT = 1.0
NU_DEFAULT = 0.3
LAMBDA_DEFAULT = E_DEFAULT * NU_DEFAULT / ((1 + NU_DEFAULT) * (1 - 2 * NU_DEFAULT))
MU_DEFAULT = E_DEFAULT / (2 * (1 + NU_DEFAULT))

LINEAR_ELASTIC = 0
NEO_HOOKEAN = 1

# Kuhn permutations and their parity (odd ones get the last two nodes swapped).
_KUHN_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))
_KUHN_ODD = (False, True, True, False, False, True)


@dataclass
class Mesh:
    """A P1 simplex mesh plus optional constraints, in the C-ABI's layout.

    coords [n_nodes, dim] float64 row-major; conn [n_elems, dim+1] int32.
    dirichlet_dofs sorted unique int32 (< N_u) with values; MPC triples
    (slave, master, offset): g_k(u) = u[slave_k] - u[master_k] - offset_k.
    """

    dim: int
    coords: np.ndarray
    conn: np.ndarray
    material: int = NEO_HOOKEAN
    lam: float = LAMBDA_DEFAULT
    mu: float = MU_DEFAULT
    dirichlet_dofs: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    dirichlet_vals: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    mpc_slave: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    mpc_master: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    mpc_offset: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))
    f_ext: Optional[np.ndarray] = None
    phase: Optional[np.ndarray] = None       # uint8 [n_elems]
    lambda_tab: Optional[np.ndarray] = None  # float64 [n_phases]
    mu_tab: Optional[np.ndarray] = None
    shape: tuple = ()                        # structured cell counts (nx, ny[, nz]) if any
    length: float = 1.0

    @property
    def n_nodes(self) -> int:
        return int(self.coords.shape[0])

    @property
    def n_elems(self) -> int:
        return int(self.conn.shape[0])

    @property
    def n_u(self) -> int:
        return self.n_nodes * self.dim

    @property
    def n_mpc(self) -> int:
        return int(self.mpc_slave.shape[0])

    @property
    def n_total(self) -> int:
        return self.n_u + self.n_mpc

    def copy_with(self, **kw) -> "Mesh":
        d = dict(self.__dict__)
        d.update(kw)
        return Mesh(**d)


# ----------------------------------------------------------------------------- meshes

def grid_tri3(nx: int, ny: int, length: float = 1.0) -> Mesh:
    """Structured [0,L]^2 Tri3 mesh (C5): (nx+1)(ny+1) nodes, 2*nx*ny elements."""
    xs = np.linspace(0.0, length, nx + 1)
    ys = np.linspace(0.0, length, ny + 1)
    X, Y = np.meshgrid(xs, ys, indexing="xy")          # [ny+1, nx+1], x fastest
    coords = np.stack([X.ravel(), Y.ravel()], axis=1).astype(np.float64)
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    a = (j * (nx + 1) + i).ravel()
    b = a + 1
    c = a + (nx + 1) + 1
    d = a + (nx + 1)
    conn = np.empty((2 * nx * ny, 3), np.int32)
    conn[0::2] = np.stack([a, b, c], axis=1)
    conn[1::2] = np.stack([a, c, d], axis=1)
    return Mesh(dim=2, coords=coords, conn=conn, shape=(nx, ny), length=length)


def delaunay_tri3(n_interior: int, n_side: int, seed: int, length: float = 1.0) -> Mesh:
    """Unstructured Tri3 mesh of [0,L]^2 (SURVEY §8(d1) structure variant): Delaunay
    triangulation (scipy.spatial) of n_interior seeded uniform points in the open square plus
    n_side + 1 equispaced points on each side, oriented counter-clockwise.  Irregular node
    degrees (the coloring / gather robustness case)."""
    from scipy.spatial import Delaunay
    rng = np.random.default_rng(seed)
    h = length / n_side
    inner = rng.uniform(0.5 * h, length - 0.5 * h, size=(n_interior, 2))
    t = np.linspace(0.0, length, n_side + 1)
    side = np.concatenate([np.stack([t, np.zeros_like(t)], 1), np.stack([t, np.full_like(t, length)], 1),
                           np.stack([np.zeros_like(t[1:-1]), t[1:-1]], 1),
                           np.stack([np.full_like(t[1:-1], length), t[1:-1]], 1)])
    coords = np.ascontiguousarray(np.concatenate([side, inner]), np.float64)
    conn = Delaunay(coords).simplices.astype(np.int32)
    X = coords[conn]
    det = ((X[:, 1, 0] - X[:, 0, 0]) * (X[:, 2, 1] - X[:, 0, 1])
           - (X[:, 2, 0] - X[:, 0, 0]) * (X[:, 1, 1] - X[:, 0, 1]))
    flip = det < 0
    conn[flip, 1], conn[flip, 2] = conn[flip, 2].copy(), conn[flip, 1].copy()
    return Mesh(dim=2, coords=coords, conn=np.ascontiguousarray(conn), length=length)


def delaunay_tet4(n_interior: int, n_side: int, seed: int, length: float = 1.0) -> Mesh:
    """Unstructured Tet4 mesh of [0,L]^3 (the "general 3D mesh" of PAPER.md App. A):
    Delaunay tetrahedralization (scipy.spatial / qhull) of n_interior seeded uniform points in
    the open cube plus the (n_side+1)^3 - (n_side-1)^3 nodes of a regular grid on its surface
    (so each boundary plane is exactly a coordinate plane: the roller BCs of C15 apply), every
    tet oriented to det J > 0.  Node degrees vary (interior ~ 13-40 neighbours), unlike the
    Kuhn meshes' uniform 14: the high-degree gather, fallback and capacity paths run."""
    from scipy.spatial import Delaunay
    rng = np.random.default_rng(seed)
    h = length / n_side
    t = np.linspace(0.0, length, n_side + 1)
    Z, Y, X = np.meshgrid(t, t, t, indexing="ij")
    grid = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    on = ((grid == 0.0) | (grid == length)).any(axis=1)
    inner = rng.uniform(0.5 * h, length - 0.5 * h, size=(n_interior, 3))
    coords = np.ascontiguousarray(np.concatenate([grid[on], inner]), np.float64)
    conn = Delaunay(coords).simplices.astype(np.int32)
    X = coords[conn]
    e = X[:, 1:, :] - X[:, :1, :]
    det = np.linalg.det(e)
    # qhull may emit (near-)flat tets spanned by four coplanar surface nodes: drop them (their
    # volume is zero, so the rest still tiles the cube; the test suite checks sum vol = L^3)
    keep = np.abs(det) > 1e-10 * h ** 3
    conn, det = conn[keep], det[keep]
    flip = det < 0
    conn[flip, 2], conn[flip, 3] = conn[flip, 3].copy(), conn[flip, 2].copy()
    used = np.unique(conn)
    if len(used) != len(coords):      # drop nodes only flat tets touched (none in practice)
        remap = np.full(len(coords), -1, np.int64)
        remap[used] = np.arange(len(used))
        coords, conn = coords[used], remap[conn].astype(np.int32)
    return Mesh(dim=3, coords=np.ascontiguousarray(coords), conn=np.ascontiguousarray(conn),
                length=length)


def grid_tet4(nx: int, ny: int, nz: int, length: float = 1.0, z0: int = 0,
              nz_total: Optional[int] = None) -> Mesh:
    """Structured Kuhn Tet4 mesh (C6) of the box [0,L]x[0,L]x[0,L*nz_total/nz_total].

    With z0/nz_total the mesh is the z-slab of cells [z0, z0+nz) of an
    nx*ny*nz_total grid (node ids local to the slab, coordinates global): used by
    the multi-GPU element partition.
    """
    nzt = nz if nz_total is None else nz_total
    xs = np.linspace(0.0, length, nx + 1)
    ys = np.linspace(0.0, length, ny + 1)
    zs = np.linspace(0.0, length, nzt + 1)[z0:z0 + nz + 1]
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")    # x fastest
    coords = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1).astype(np.float64)
    sx, sy = 1, nx + 1
    sz = (nx + 1) * (ny + 1)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    v0 = (k * sz + j * sy + i * sx).ravel().astype(np.int64)
    step = (sx, sy, sz)
    n_cells = v0.shape[0]
    conn = np.empty((n_cells, 6, 4), np.int32)
    for t, (perm, odd) in enumerate(zip(_KUHN_PERMS, _KUHN_ODD)):
        n1 = v0 + step[perm[0]]
        n2 = n1 + step[perm[1]]
        n3 = n2 + step[perm[2]]
        if odd:
            n2, n3 = n3, n2
        conn[:, t, 0] = v0
        conn[:, t, 1] = n1
        conn[:, t, 2] = n2
        conn[:, t, 3] = n3
    return Mesh(dim=3, coords=coords, conn=conn.reshape(-1, 4), shape=(nx, ny, nz),
                length=length)


def boundary_node_mask(mesh: Mesh, length: Optional[float] = None) -> np.ndarray:
    """Nodes lying on the boundary planes of the structured box (by index, exact)."""
    L = mesh.length if length is None else length
    tol = 1e-12 * L
    on = np.zeros(mesh.n_nodes, bool)
    for c in range(mesh.dim):
        x = mesh.coords[:, c]
        on |= (np.abs(x) <= tol) | (np.abs(x - L) <= tol)
    return on


def perturb(mesh: Mesh, a: float, seed: int, h: Optional[float] = None) -> Mesh:
    """C16: jitter interior nodes by U(-a*h, a*h) per coordinate; boundary nodes fixed."""
    if h is None:
        h = mesh.length / max(mesh.shape)
    rng = np.random.default_rng(seed)
    interior = ~boundary_node_mask(mesh)
    jit = rng.uniform(-a * h, a * h, size=mesh.coords.shape)
    coords = mesh.coords.copy()
    coords[interior] += jit[interior]
    return mesh.copy_with(coords=coords)


def renumber_nodes(mesh: Mesh, seed: int) -> Mesh:
    """Random node permutation (the 'shuffled numbering' variant)."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(mesh.n_nodes)          # new id of old node i is perm[i]
    coords = np.empty_like(mesh.coords)
    coords[perm] = mesh.coords
    conn = perm[mesh.conn].astype(np.int32)
    return mesh.copy_with(coords=coords, conn=conn)


# ----------------------------------------------------------------------- constraints

def _nodes_at(mesh: Mesh, comp: int, value: float) -> np.ndarray:
    tol = 1e-12 * mesh.length
    return np.nonzero(np.abs(mesh.coords[:, comp] - value) <= tol)[0]


def roller_bc(mesh: Mesh, eps: float) -> Mesh:
    """C15 roller uniaxial stretch: u_x=0 on x=0; u_y=0 on y=0; (u_z=0 on z=0);
    u_x = eps*L on x=L.  Other DOFs free."""
    m, L = mesh.dim, mesh.length
    dofs, vals = [], []
    for c in range(m):
        nodes = _nodes_at(mesh, c, 0.0)
        dofs.append(nodes * m + c)
        vals.append(np.zeros(nodes.shape[0]))
    nodes = _nodes_at(mesh, 0, L)
    dofs.append(nodes * m + 0)
    vals.append(np.full(nodes.shape[0], eps * L))
    dofs = np.concatenate(dofs)
    vals = np.concatenate(vals)
    order = np.argsort(dofs, kind="stable")
    dofs, vals = dofs[order], vals[order]
    uniq, first = np.unique(dofs, return_index=True)
    return mesh.copy_with(dirichlet_dofs=uniq.astype(np.int32),
                          dirichlet_vals=vals[first].astype(np.float64))


def roller_symmetry_bc(mesh: Mesh) -> Mesh:
    """Symmetry rollers only: u_x=0 on x=0, u_y=0 on y=0 (, u_z=0 on z=0) — the traction
    problem of PAPER.md §6.1 without the prescribed stretch."""
    m = mesh.dim
    dofs = np.concatenate([_nodes_at(mesh, c, 0.0) * m + c for c in range(m)])
    uniq = np.unique(dofs)
    return mesh.copy_with(dirichlet_dofs=uniq.astype(np.int32),
                          dirichlet_vals=np.zeros(uniq.shape[0]))


def boundary_facets(mesh: Mesh, comp: int, value: float) -> np.ndarray:
    """Facets (Line2 in 2D, Tri3 in 3D; [n][dim] node ids) of the elements lying on the
    plane X_comp = value: element faces whose nodes all sit on it (each boundary face belongs
    to exactly one element)."""
    on = np.zeros(mesh.n_nodes, bool)
    on[_nodes_at(mesh, comp, value)] = True
    d = mesh.dim
    out = []
    for drop in range(d + 1):
        face = np.delete(mesh.conn, drop, axis=1)
        out.append(face[on[face].all(axis=1)])
    return np.ascontiguousarray(np.concatenate(out), dtype=np.int32)


def clamped_bc(mesh: Mesh, eps: float) -> Mesh:
    """C15 clamped variant: u = 0 on x=0; u = (eps*L, 0[, 0]) on x=L."""
    m, L = mesh.dim, mesh.length
    left = _nodes_at(mesh, 0, 0.0)
    right = _nodes_at(mesh, 0, L)
    dofs = np.concatenate([left[:, None] * m + np.arange(m), right[:, None] * m + np.arange(m)])
    vals = np.concatenate([np.zeros((left.size, m)),
                           np.tile(np.r_[eps * L, np.zeros(m - 1)], (right.size, 1))])
    dofs, vals = dofs.ravel(), vals.ravel()
    order = np.argsort(dofs, kind="stable")
    return mesh.copy_with(dirichlet_dofs=dofs[order].astype(np.int32),
                          dirichlet_vals=vals[order].astype(np.float64))


def periodic_mpc(mesh: Mesh, eps_hat: np.ndarray) -> Mesh:
    """C13 periodic constraints on a structured 2D nx*ny grid.

    Left<->right pairs for every row j in [0, ny] (slave x=L, master x=0);
    bottom<->top pairs for columns i in [0, nx-1] (slave y=L, master y=0).
    Each pair gives one constraint per component with offset
    b = eps_hat @ (X_s - X_m) (total-displacement form of u = eps_hat x + u~).
    Node 0 is pinned (u = 0, Dirichlet) to remove rigid translation.
    """
    assert mesh.dim == 2 and len(mesh.shape) == 2
    nx, ny = mesh.shape
    m = 2
    slaves, masters = [], []
    for j in range(ny + 1):
        slaves.append(j * (nx + 1) + nx)
        masters.append(j * (nx + 1) + 0)
    for i in range(nx):
        slaves.append(ny * (nx + 1) + i)
        masters.append(i)
    slaves = np.asarray(slaves, np.int64)
    masters = np.asarray(masters, np.int64)
    dX = mesh.coords[slaves] - mesh.coords[masters]          # [pairs, 2]
    off = dX @ np.asarray(eps_hat, np.float64).T              # [pairs, 2]
    s_dof = (slaves[:, None] * m + np.arange(m)).ravel()
    m_dof = (masters[:, None] * m + np.arange(m)).ravel()
    return mesh.copy_with(mpc_slave=s_dof.astype(np.int32), mpc_master=m_dof.astype(np.int32),
                          mpc_offset=off.ravel().astype(np.float64),
                          dirichlet_dofs=np.array([0, 1], np.int32),
                          dirichlet_vals=np.zeros(2))


def two_phase(mesh: Mesh, radius: float, lam_mu_matrix, lam_mu_incl) -> Mesh:
    """Per-element phase table: elements whose first node lies within `radius` of the
    cell centre are phase 1 (synthetic stand-in for the P:490 inclusion cell)."""
    c = mesh.coords[mesh.conn[:, 0]]
    ctr = np.full(mesh.dim, 0.5 * mesh.length)
    phase = (np.linalg.norm(c - ctr, axis=1) < radius).astype(np.uint8)
    return mesh.copy_with(phase=phase,
                          lambda_tab=np.array([lam_mu_matrix[0], lam_mu_incl[0]], np.float64),
                          mu_tab=np.array([lam_mu_matrix[1], lam_mu_incl[1]], np.float64))


# ---------------------------------------------------------------------------- states

def affine_field(mesh: Mesh, A: np.ndarray, c: Optional[np.ndarray] = None) -> np.ndarray:
    """u(X) = A X + c sampled at the nodes, flattened node-major (DOF = node*m+comp)."""
    u = mesh.coords @ np.asarray(A, np.float64).T
    if c is not None:
        u = u + np.asarray(c, np.float64)
    return np.ascontiguousarray(u.ravel())


def generic_state(mesh: Mesh, seed: int, eps: float = 0.05, noise: float = 0.01,
                  h: Optional[float] = None) -> np.ndarray:
    """§8(c4): affine stretch (eps) plus U(-noise*h, noise*h) per DOF, multipliers U(-1,1)."""
    if h is None:  # structured: the cell size; unstructured: the equivalent grid spacing
        if mesh.shape:
            h = mesh.length / max(mesh.shape)
        else:
            per_cell = 2 if mesh.dim == 2 else 6
            h = mesh.length * (per_cell / max(mesh.n_elems, 1)) ** (1.0 / mesh.dim)
    rng = np.random.default_rng(seed)
    A = np.zeros((mesh.dim, mesh.dim))
    A[0, 0] = eps
    u = affine_field(mesh, A)
    u += rng.uniform(-noise * h, noise * h, size=u.shape)
    if mesh.n_mpc:
        u = np.concatenate([u, rng.uniform(-1.0, 1.0, size=mesh.n_mpc)])
    return u


def random_direction(n: int, seed: int) -> np.ndarray:
    """v ~ U(-1, 1) (§8(c4))."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=n)


def lift(mesh: Mesh, z: Optional[np.ndarray] = None) -> np.ndarray:
    """z with z[D] = g (the lift of the reduced functional)."""
    out = np.zeros(mesh.n_total) if z is None else np.array(z, np.float64, copy=True)
    out[mesh.dirichlet_dofs] = mesh.dirichlet_vals
    return out


# -------------------------------------------------------------------- named configs

def config_mesh(cfg: int, n: Optional[int] = None, perturbed: bool = True) -> Mesh:
    """BASELINE.json configs as concrete synthetic meshes.

    cfg 1: 2D LE 8x8 unit square; cfg 2: 2D NH 706^2 plate (roller eps=0.1);
    cfg 3: 3D NH 150^3 Kuhn block (roller eps=0.05); cfg 4: 3D NH 255x255x256 (seed 14);
    cfg 5: 2D LE n^2 with periodic MPC.  `n` overrides the size.
    """
    if cfg == 1:
        m = grid_tri3(8, 8)
        if perturbed:
            m = perturb(m, 0.2, seed=11)
        return m.copy_with(material=LINEAR_ELASTIC)
    if cfg == 2:
        k = 706 if n is None else n
        m = grid_tri3(k, k)
        if perturbed:
            m = perturb(m, 0.1, seed=12)
        return roller_bc(m.copy_with(material=NEO_HOOKEAN), eps=0.1)
    if cfg == 3:
        k = 150 if n is None else n
        m = grid_tet4(k, k, k)
        if perturbed:
            m = perturb(m, 0.1, seed=13)
        return roller_bc(m.copy_with(material=NEO_HOOKEAN), eps=0.05)
    if cfg == 4:  # n x n x (n + 1) cells, like 255 x 255 x 256 (z-slabs of 256 / P, §8(e))
        m = grid_tet4(255, 255, 256) if n is None else grid_tet4(n, n, n + 1)
        if perturbed:
            m = perturb(m, 0.1, seed=14)
        return roller_bc(m.copy_with(material=NEO_HOOKEAN), eps=0.05)
    if cfg == 5:
        k = 70 if n is None else n
        m = grid_tri3(k, k)
        if perturbed:
            m = perturb(m, 0.1, seed=15)
        eps_hat = np.array([[0.01, 0.005], [0.005, -0.003]])
        return periodic_mpc(m.copy_with(material=LINEAR_ELASTIC), eps_hat)
    raise ValueError(f"unknown config {cfg}")
