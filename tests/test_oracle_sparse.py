"""Pins for the oracle's pattern, coloring, Alg. 2 assembly, SpMV, CG and Newton.

Pinned against SPEC/paper worked examples (tests/golden/spec_examples.json), closed-form
nnz counts, the dense Hessian (entries off the pattern exactly 0; colored CSR equals the
dense Hessian bitwise), networkx's greedy coloring in ascending order, scipy.sparse,
numpy.linalg.solve, and the closed-form homogeneous Newton solutions.
"""
import json
import os

import networkx as nx
import numpy as np
import pytest
import scipy.sparse as sp

import fem_inputs as fi
from tests import _textbook as tb

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def csr_rows(rp):
    return np.repeat(np.arange(len(rp) - 1), np.diff(rp))


def nnz_closed_form(mesh):
    """nnz = m^2 (N_nodes + 2 edges) with the closed-form edge counts."""
    m = mesh.dim
    if m == 2:
        nx_, ny_ = mesh.shape
        edges = nx_ * (ny_ + 1) + ny_ * (nx_ + 1) + nx_ * ny_
    else:
        a, b, c = mesh.shape
        edges = (a * (b + 1) * (c + 1) + (a + 1) * b * (c + 1) + (a + 1) * (b + 1) * c
                 + a * b * (c + 1) + a * (b + 1) * c + (a + 1) * b * c + a * b * c)
    return m * m * (mesh.n_nodes + 2 * edges)


# ------------------------------------------------------------------------------ pattern

def test_pattern_spec_examples(oracle_mod):
    one = fi.Mesh(dim=2, coords=np.array([[0., 0.], [1., 0.], [0., 1.]]),
                  conn=np.array([[0, 1, 2]], np.int32))
    two = fi.Mesh(dim=2, coords=np.array([[0., 0.], [1., 0.], [1., 1.], [0., 1.]]),
                  conn=np.array([[0, 1, 2], [0, 2, 3]], np.int32))
    # m = dim = 2 here: every m=1 entry becomes a 2x2 block
    assert len(oracle_mod.Oracle(one).sparsity()[1]) == 4 * GOLD["pattern_single_tri3_m1"]["nnz_m1"]
    assert len(oracle_mod.Oracle(two).sparsity()[1]) == 4 * GOLD["pattern_two_tri3_m1"]["nnz_m1"]


@pytest.mark.parametrize("mesh", [fi.grid_tri3(8, 8), fi.grid_tri3(13, 5), fi.grid_tet4(6, 6, 6),
                                  fi.grid_tet4(3, 5, 4)])
def test_pattern_closed_form_sorted_symmetric(oracle_mod, mesh):
    rp, ci = oracle_mod.Oracle(mesh).sparsity()
    assert rp[-1] == nnz_closed_form(mesh)
    if mesh.shape == (8, 8):
        assert rp[-1] == 1988
    if mesh.shape == (6, 6, 6):
        assert rp[-1] == 9 * 4051
    for i in range(len(rp) - 1):
        assert np.all(np.diff(ci[rp[i]:rp[i + 1]]) > 0)
    A = sp.csr_matrix((np.ones(len(ci)), ci, rp))
    assert (A - A.T).nnz == 0


@pytest.mark.parametrize("material", [0, 1])
def test_dense_hessian_vanishes_off_pattern(oracle_mod, material):
    m = fi.perturb(fi.grid_tri3(5, 4), 0.2, 1).copy_with(material=material)
    o = oracle_mod.Oracle(m)
    H = o.dense_hessian(fi.generic_state(m, 1))
    rp, ci = o.sparsity()
    H[csr_rows(rp), ci] = 0.0
    assert np.all(H == 0.0)


def test_augmented_pattern(oracle_mod):
    m = fi.config_mesh(5, n=6)
    o = oracle_mod.Oracle(m)
    rp, ci = o.sparsity()
    base = oracle_mod.Oracle(m.copy_with(mpc_slave=m.mpc_slave[:0], mpc_master=m.mpc_master[:0],
                                         mpc_offset=m.mpc_offset[:0])).sparsity()
    assert rp[-1] == base[0][-1] + 4 * m.n_mpc          # B and B^T blocks, empty 0 block
    H = o.dense_hessian(fi.generic_state(m, 2))
    pat = np.zeros_like(H, bool)
    pat[csr_rows(rp), ci] = True
    assert np.all(H[~pat] == 0.0)
    assert not pat[m.n_u:, m.n_u:].any()                # SPEC S:393 empty multiplier block


# ----------------------------------------------------------------------------- coloring

def column_intersection_graph(rp, ci):
    n = len(rp) - 1
    G = nx.Graph()
    G.add_nodes_from(range(n))
    for i in range(n):
        cols = ci[rp[i]:rp[i + 1]]
        for a in range(len(cols)):
            for b in range(a + 1, len(cols)):
                G.add_edge(int(cols[a]), int(cols[b]))
    return G


def assert_valid(rp, ci, colors):
    for i in range(len(rp) - 1):
        c = colors[ci[rp[i]:rp[i + 1]]]
        assert len(np.unique(c)) == len(c)          # SPEC S:409 validity


def test_coloring_spec_examples(oracle_mod):
    n = 6
    tri = sp.diags([np.ones(n - 1), np.ones(n), np.ones(n - 1)], [-1, 0, 1]).tocsr()
    col, nc = oracle_mod.color(tri.indptr, tri.indices)
    assert nc == GOLD["color_tridiagonal_6"]["n_colors"]
    assert col.tolist() == GOLD["color_tridiagonal_6"]["colors"]
    d = sp.identity(7).tocsr()
    assert oracle_mod.color(d.indptr, d.indices)[1] == GOLD["color_diagonal"]["n_colors"]
    full = sp.csr_matrix(np.ones((5, 5)))
    col, nc = oracle_mod.color(full.indptr, full.indices)
    assert nc == 5 and sorted(col.tolist()) == list(range(5))


@pytest.mark.parametrize("mesh", [fi.grid_tri3(8, 8), fi.grid_tri3(9, 9), fi.grid_tet4(4, 4, 4),
                                  fi.renumber_nodes(fi.grid_tri3(7, 6), 21),
                                  fi.config_mesh(5, n=8), fi.delaunay_tri3(150, 8, 3),
                                  fi.delaunay_tet4(40, 3, 5)])
def test_coloring_equals_networkx_ordered_greedy(oracle_mod, mesh):
    o = oracle_mod.Oracle(mesh)
    rp, ci = o.sparsity()
    colors, nc = o.colors()
    G = column_intersection_graph(rp, ci)
    ref = nx.greedy_color(G, strategy=lambda g, c: sorted(g.nodes()))
    assert all(colors[j] == ref[j] for j in range(len(colors)))
    assert nc == max(ref.values()) + 1
    assert_valid(rp, ci, colors)


def test_color_counts_size_independent(oracle_mod):
    counts2 = [oracle_mod.Oracle(fi.grid_tri3(n, n)).colors()[1] for n in (8, 16, 32)]
    assert counts2 == [18, 18, 18]                       # 9 node colors x m = 2
    # m = 3 Kuhn tets: 87 for n >= 12; paper range 80-90
    c3 = oracle_mod.Oracle(fi.grid_tet4(12, 12, 12)).colors()[1]
    assert c3 == 87
    assert GOLD["color_range_3d_tet4"]["lo"] <= c3 <= GOLD["color_range_3d_tet4"]["hi"]


# --------------------------------------------------------------------------- assembly

CASES = [("le", fi.perturb(fi.grid_tri3(8, 8), 0.2, 11).copy_with(material=0), False),
         ("nh", fi.perturb(fi.grid_tri3(8, 8), 0.2, 11).copy_with(material=1), False),
         ("nh-bc", fi.roller_bc(fi.perturb(fi.grid_tri3(8, 8), 0.2, 11).copy_with(material=1), 0.1), True),
         ("nh3d-bc", fi.roller_bc(fi.perturb(fi.grid_tet4(3, 3, 3), 0.1, 2), 0.05), True),
         ("mpc", fi.config_mesh(5, n=6), False)]


@pytest.mark.parametrize("name,mesh,bc", CASES, ids=[c[0] for c in CASES])
def test_alg2_equals_dense_hessian_bitwise(oracle_mod, name, mesh, bc):
    o = oracle_mod.Oracle(mesh)
    z = fi.lift(mesh, fi.generic_state(mesh, 3)) if bc else fi.generic_state(mesh, 3)
    rp, ci = o.sparsity()
    vals = o.assemble_alg2(z, bc=bc)
    H = o.dense_hessian(z, bc=bc)
    assert np.array_equal(vals, H[csr_rows(rp), ci])
    if bc:  # masked operator = P_f K P_f + P_D (reading C12)
        K = o.dense_hessian(z)
        Pf = np.ones(mesh.n_total); Pf[mesh.dirichlet_dofs] = 0.0
        ref = Pf[:, None] * K * Pf[None, :] + np.diag(1 - Pf)
        assert np.array_equal(H, ref)
    ve = o.assemble_elem(z, bc=bc)
    assert np.abs(ve - vals).max() <= 1e-14 * np.abs(vals).max()
    rows = np.array([0, 5, mesh.n_total // 2, mesh.n_total - 1])
    packed = o.csr_rows(z, rows, rp, ci, bc=bc)
    ref = np.concatenate([ve[rp[r]:rp[r + 1]] for r in rows])
    assert np.abs(packed - ref).max() <= 1e-15 * np.abs(vals).max()


def test_row_sampled_residual_hvp(oracle_mod):
    m = fi.roller_bc(fi.perturb(fi.grid_tet4(3, 4, 3), 0.1, 3), 0.05)
    o = oracle_mod.Oracle(m)
    z = fi.lift(m, fi.generic_state(m, 4))
    v = fi.random_direction(m.n_total, 5)
    rows = np.random.default_rng(0).choice(m.n_total, 40, replace=False)
    for bc in (False, True):
        assert np.abs(o.residual_rows(z, rows, bc) - o.residual(z, bc)[rows]).max() < 1e-16
        assert np.abs(o.hvp_rows(z, v, rows, bc) - o.hvp(z, v, bc)[rows]).max() < 1e-15


def test_spmv_matches_scipy_and_hvp(oracle_mod):
    m = fi.perturb(fi.grid_tri3(8, 8), 0.2, 11)
    o = oracle_mod.Oracle(m)
    z = fi.generic_state(m, 1)
    rp, ci = o.sparsity()
    vals = o.assemble_alg2(z)
    x = fi.random_direction(m.n_total, 2)
    y = oracle_mod.spmv(rp, ci, vals, x)
    ref = sp.csr_matrix((vals, ci, rp)) @ x
    assert np.abs(y - ref).max() < 1e-14 * np.abs(ref).max()
    assert np.abs(y - o.hvp(z, x)).max() < 1e-13 * np.abs(ref).max()


# ------------------------------------------------------------------------------ solvers

def test_cg_spec_examples(oracle_mod):
    g = GOLD["cg_2x2"]
    A = sp.csr_matrix(np.array(g["A"], float))
    x, rep = oracle_mod.cg_csr(A.indptr, A.indices, A.data, np.array(g["b"], float), rtol=1e-15)
    assert rep["status"] == 0
    assert np.abs(x - np.array(g["x"])).max() < 1e-15
    I = sp.identity(4).tocsr()
    b = np.arange(1.0, 5.0)
    x, rep = oracle_mod.cg_csr(I.indptr, I.indices, I.data, b)
    assert rep["iters"] == 1 and np.array_equal(x, b)
    x, rep = oracle_mod.cg_csr(I.indptr, I.indices, I.data, np.zeros(4))
    assert rep["iters"] == 0 and np.all(x == 0)
    rng = np.random.default_rng(0)
    Q = rng.standard_normal((50, 50))
    S = Q @ Q.T + 50 * np.eye(50)
    Ssp = sp.csr_matrix(S)
    b = rng.standard_normal(50)
    x, rep = oracle_mod.cg_csr(Ssp.indptr, Ssp.indices, Ssp.data, b, rtol=1e-14)
    assert np.abs(x - np.linalg.solve(S, b)).max() < 1e-9
    # breakdown on an indefinite matrix
    N = sp.csr_matrix(np.diag([1.0, -1.0]))
    _, rep = oracle_mod.cg_csr(N.indptr, N.indices, N.data, np.array([1.0, 1.0]))
    assert rep["status"] == 5


def test_cg_matrix_free_equals_direct_solve(oracle_mod):
    m = fi.roller_bc(fi.perturb(fi.grid_tri3(6, 6), 0.2, 3).copy_with(material=1), 0.1)
    o = oracle_mod.Oracle(m)
    z = fi.lift(m, fi.generic_state(m, 1))
    b = fi.random_direction(m.n_total, 2); b[m.dirichlet_dofs] = 0.0
    x, rep = o.cg(b, op=0, z=z, rtol=1e-14)
    H = o.dense_hessian(z, bc=True)
    assert rep["status"] == 0
    assert np.abs(x - np.linalg.solve(H, b)).max() < 1e-10 * np.abs(x).max()


def test_newton_linear_elastic_one_iteration(oracle_mod):
    m = fi.roller_bc(fi.perturb(fi.grid_tri3(6, 6), 0.2, 3).copy_with(material=0), 0.1)
    z, rep = oracle_mod.Oracle(m).newton(fi.lift(m), cg_rtol=1e-14)
    assert rep["status"] == 0 and rep["iters"] == GOLD["newton_quadratic_one_step"]["iters"]


@pytest.mark.parametrize("dim,eps", [(2, 0.1), (3, 0.05)])
def test_newton_roller_homogeneous_solution(oracle_mod, dim, eps):
    # C15: the roller stretch has a homogeneous FE solution u = (F - I) X on ANY P1 mesh
    base = fi.perturb(fi.grid_tri3(8, 8), 0.2, 11) if dim == 2 else fi.perturb(fi.grid_tet4(3, 3, 3), 0.1, 2)
    m = fi.roller_bc(base.copy_with(material=1), eps)
    o = oracle_mod.Oracle(m)
    z, rep = o.newton(fi.lift(m), cg_rtol=1e-13)
    assert rep["status"] == 0 and rep["iters"] <= 8
    U = z.reshape(-1, dim)
    A, *_ = np.linalg.lstsq(m.coords, U, rcond=None)       # U = X A  (A = (F - I)^T)
    assert np.abs(m.coords @ A - U).max() < 1e-12
    F = A.T + np.eye(dim)
    assert abs(F[0, 0] - (1 + eps)) < 1e-12
    assert np.abs(F - np.diag(np.diag(F))).max() < 1e-12
    s = F[1, 1]
    assert all(abs(F[k, k] - s) < 1e-12 for k in range(1, dim))
    # s makes the homogeneous energy stationary: d/ds Psi(diag(1+eps, s, ..)) = 0
    def Psi(t):
        G = np.diag([eps] + [t - 1.0] * (dim - 1))
        return o.energy(fi.affine_field(m, G))
    h = 1e-5
    assert abs((Psi(s + h) - Psi(s - h)) / (2 * h)) < 1e-9
    assert 0.9 < s < 1.0


def test_periodic_homogeneous_solution(oracle_mod):
    # homogeneous material + periodic BC with macro strain eps_hat => u = eps_hat X exactly
    m = fi.config_mesh(5, n=8)
    o = oracle_mod.Oracle(m)
    rp, ci = o.sparsity()
    z0 = fi.lift(m)
    Kc = sp.csr_matrix((o.assemble_alg2(z0, bc=True), ci, rp)).toarray()
    r0 = o.residual(z0, bc=True)
    z = z0 + np.linalg.solve(Kc, -r0)
    eps_hat = np.array([[0.01, 0.005], [0.005, -0.003]])
    ref = fi.affine_field(m, eps_hat)
    assert np.abs(z[:m.n_u] - ref).max() < 1e-14
    assert np.abs(o.residual(z, bc=True)).max() < 1e-14
    assert np.abs(tb.constraint_matrix(m) @ z[:m.n_u] - m.mpc_offset).max() < 1e-15
