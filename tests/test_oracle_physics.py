"""Pins for the oracle's energy, residual and HVP (SURVEY §8(c5) checklist).

Each test pins the oracle to something other than itself: closed forms of the
densities on single elements, a textbook B^T D B stiffness (tests/_textbook.py),
rigid-body and patch-test invariants, central finite differences, symmetry,
the small-strain limit NH -> LE, and the LE null space dimension.
"""
import numpy as np
import pytest

import fem_inputs as fi
from tests import _textbook as tb

LAM, MU = fi.LAMBDA_DEFAULT, fi.MU_DEFAULT


def unit_simplex(dim, material, lam=LAM, mu=MU):
    if dim == 2:
        X = np.array([[0., 0.], [1., 0.], [0., 1.]])
    else:
        X = np.array([[0., 0., 0.], [1., 0., 0.], [0., 1., 0.], [0., 0., 1.]])
    return fi.Mesh(dim=dim, coords=X, conn=np.arange(dim + 1, dtype=np.int32)[None],
                   material=material, lam=lam, mu=mu)


def energy_of_H(oracle_mod, dim, material, H, lam=LAM, mu=MU):
    m = unit_simplex(dim, material, lam, mu)
    u = fi.affine_field(m, H)
    vol = 0.5 if dim == 2 else 1.0 / 6.0
    return oracle_mod.Oracle(m).energy(u) / vol


def small_mesh(dim, material, perturbed=True, seed=7):
    m = fi.grid_tri3(6, 5) if dim == 2 else fi.grid_tet4(3, 3, 2)
    if perturbed:
        m = fi.perturb(m, 0.2 if dim == 2 else 0.1, seed)
    return m.copy_with(material=material)


def rotation(dim, angle):
    c, s = np.cos(angle), np.sin(angle)
    if dim == 2:
        return np.array([[c, -s], [s, c]])
    R1 = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.]])
    R2 = np.array([[1., 0, 0], [0, np.cos(0.4), -np.sin(0.4)], [0, np.sin(0.4), np.cos(0.4)]])
    return R1 @ R2


# ------------------------------------------------------------------------ energy density

@pytest.mark.parametrize("dim", [2, 3])
def test_le_closed_forms(oracle_mod, dim):
    e, g = 1e-3, 0.02
    H = np.zeros((dim, dim)); H[0, 0] = e
    # uniaxial strain: psi = (lambda + 2 mu) e^2 / 2
    assert abs(energy_of_H(oracle_mod, dim, 0, H) - 0.5 * (LAM + 2 * MU) * e * e) < 1e-15 * 1e-6
    H = np.zeros((dim, dim)); H[0, 1] = g
    # simple shear: psi = mu gamma^2 / 2
    assert abs(energy_of_H(oracle_mod, dim, 0, H) - 0.5 * MU * g * g) < 1e-18
    # general H against the textbook Voigt form 1/2 eps^T D eps
    H = np.random.default_rng(1).uniform(-0.1, 0.1, (dim, dim))
    ref = tb.strain_energy_density(H, LAM, MU)
    assert abs(energy_of_H(oracle_mod, dim, 0, H) - ref) < 1e-14 * ref


def test_nh_closed_forms(oracle_mod):
    # SPEC S:643 (reading C1): psi = mu/2 (I1 - d - 2 ln J) + lambda/2 (ln J)^2
    # F = diag(2, 1), mu = lambda = 1: I1 = 5, J = 2
    H = np.array([[1.0, 0.0], [0.0, 0.0]])
    ref = 0.5 * (5 - 2 - 2 * np.log(2.0)) + 0.5 * np.log(2.0) ** 2
    assert abs(energy_of_H(oracle_mod, 2, 1, H, 1.0, 1.0) - ref) < 1e-15
    # isochoric simple shear (J = 1): psi = mu gamma^2 / 2 for any lambda
    for dim in (2, 3):
        H = np.zeros((dim, dim)); H[0, dim - 1] = 0.3
        assert abs(energy_of_H(oracle_mod, dim, 1, H, 7.0, 0.8) - 0.5 * 0.8 * 0.09) < 1e-15
    # pure dilation F = a I in 3D: I1 = 3a^2, ln J = 3 ln a
    a = 1.1
    ref = 0.25 * (3 * a * a - 3 - 6 * np.log(a)) + 1.0 * (3 * np.log(a)) ** 2
    assert abs(energy_of_H(oracle_mod, 3, 1, (a - 1) * np.eye(3), 2.0, 0.5) - ref) < 1e-15


@pytest.mark.parametrize("dim", [2, 3])
def test_nh_invariances(oracle_mod, dim):
    assert energy_of_H(oracle_mod, dim, 1, np.zeros((dim, dim))) == 0.0       # F = I
    R = rotation(dim, 0.7)
    assert abs(energy_of_H(oracle_mod, dim, 1, R - np.eye(dim))) < 1e-15      # frame invariance
    rng = np.random.default_rng(3)
    for _ in range(20):                                                      # psi >= 0
        H = rng.uniform(-0.3, 0.3, (dim, dim))
        assert energy_of_H(oracle_mod, dim, 1, H) >= 0.0
    # small-strain limit NH -> LE: relative difference O(|H|)
    H = rng.uniform(-1, 1, (dim, dim))
    for t, bound in ((1e-3, 5e-3), (1e-5, 5e-5)):
        le = energy_of_H(oracle_mod, dim, 0, t * H)
        nh = energy_of_H(oracle_mod, dim, 1, t * H)
        assert abs(nh - le) / le < bound


def test_inverted_element_rejected(oracle_mod):
    with pytest.raises(oracle_mod.OracleError) as ei:
        energy_of_H(oracle_mod, 2, 1, np.array([[-2.0, 0.0], [0.0, 0.0]]))
    assert ei.value.status == 3


@pytest.mark.parametrize("dim", [2, 3])
def test_energy_of_affine_field_integrates_exactly(oracle_mod, dim):
    m = small_mesh(dim, 0)
    A = np.random.default_rng(5).uniform(-0.1, 0.1, (dim, dim))
    E = oracle_mod.Oracle(m).energy(fi.affine_field(m, A))
    ref = tb.strain_energy_density(A, LAM, MU)            # |Omega| = 1
    assert abs(E - ref) < 1e-14 * ref
    mn = m.copy_with(material=1)
    En = oracle_mod.Oracle(mn).energy(fi.affine_field(m, A))
    assert abs(En - energy_of_H(oracle_mod, dim, 1, A)) < 1e-14 * En


# ----------------------------------------------------------------------------- residual

@pytest.mark.parametrize("dim", [2, 3])
def test_le_residual_is_textbook_K_u(oracle_mod, dim):
    m = small_mesh(dim, 0)
    K = tb.stiffness(m)
    u = fi.generic_state(m, 1)
    r = oracle_mod.Oracle(m).residual(u)
    ref = K @ u
    assert np.abs(r - ref).max() < 1e-14 * np.abs(ref).max() * 10


@pytest.mark.parametrize("dim,material", [(2, 0), (2, 1), (3, 0), (3, 1)])
def test_rigid_motion_zero_residual(oracle_mod, dim, material):
    m = small_mesh(dim, material)
    o = oracle_mod.Oracle(m)
    scale = np.abs(o.residual(fi.generic_state(m, 2))).max()
    c = np.arange(1, dim + 1) * 0.01
    if material == 0:
        W = np.zeros((dim, dim)); W[0, 1], W[1, 0] = 1e-3, -1e-3   # infinitesimal rotation
        u = fi.affine_field(m, W, c)
    else:
        u = fi.affine_field(m, rotation(dim, 0.9) - np.eye(dim), c)  # finite rotation
    assert abs(o.energy(u)) < 1e-15
    assert np.abs(o.residual(u)).max() < 1e-14 * scale * 10


@pytest.mark.parametrize("dim,material", [(2, 0), (2, 1), (3, 0), (3, 1)])
def test_patch_test_interior_residual_vanishes(oracle_mod, dim, material):
    m = small_mesh(dim, material)
    o = oracle_mod.Oracle(m)
    A = np.random.default_rng(9).uniform(-0.08, 0.08, (dim, dim))
    r = o.residual(fi.affine_field(m, A)).reshape(-1, dim)
    interior = ~fi.boundary_node_mask(m)
    scale = np.abs(r).max()
    assert scale > 1e-4
    assert np.abs(r[interior]).max() < 1e-14 * scale * 10
    # per-component sum over all nodes vanishes (translation invariance)
    assert np.abs(r.sum(axis=0)).max() < 1e-14 * scale * 10


@pytest.mark.parametrize("dim,material", [(2, 0), (2, 1), (3, 1)])
def test_residual_matches_energy_fd(oracle_mod, dim, material):
    m = small_mesh(dim, material)
    o = oracle_mod.Oracle(m)
    u = fi.generic_state(m, 4)
    r = o.residual(u)
    h = 1e-6
    rng = np.random.default_rng(0)
    for i in rng.choice(m.n_u, 8, replace=False):
        e = np.zeros_like(u); e[i] = h
        fd = (o.energy(u + e) - o.energy(u - e)) / (2 * h)
        assert abs(fd - r[i]) < 1e-8 * np.abs(r).max()


def test_residual_bc_fext_and_mpc_terms(oracle_mod):
    m = fi.config_mesh(5, n=6)
    rng = np.random.default_rng(2)
    m = m.copy_with(f_ext=rng.uniform(-1, 1, m.n_u))
    o = oracle_mod.Oracle(m)
    z = fi.generic_state(m, 3)
    r = o.residual(z)
    B = tb.constraint_matrix(m)
    u, lam = z[:m.n_u], z[m.n_u:]
    # multiplier rows: g(u) = B u - b
    assert np.abs(r[m.n_u:] - (B @ u - m.mpc_offset)).max() < 1e-15
    # displacement rows: K u + B^T lambda - f_ext
    K = tb.stiffness(m)
    ref = K @ u + B.T @ lam - m.f_ext
    assert np.abs(r[:m.n_u] - ref).max() < 1e-13 * np.abs(ref).max()
    rb = o.residual(z, bc=True)
    assert np.all(rb[m.dirichlet_dofs] == 0.0)
    keep = np.setdiff1d(np.arange(m.n_total), m.dirichlet_dofs)
    assert np.array_equal(rb[keep], r[keep])
    # energy includes lambda . g(u) - f_ext . u
    E0 = oracle_mod.Oracle(m.copy_with(f_ext=None, mpc_slave=m.mpc_slave[:0],
                                       mpc_master=m.mpc_master[:0],
                                       mpc_offset=m.mpc_offset[:0])).energy(u)
    assert abs(o.energy(z) - (E0 + lam @ (B @ u - m.mpc_offset) - m.f_ext @ u)) < 1e-14


def test_periodic_antisymmetry(oracle_mod):
    # T-res-periodic: at u = eps_hat X, r[s_k] + r[m_k] = 0 for non-corner pairs
    m = fi.config_mesh(5, n=8)
    eps_hat = np.array([[0.01, 0.005], [0.005, -0.003]])
    z = np.concatenate([fi.affine_field(m, eps_hat), np.zeros(m.n_mpc)])
    r = oracle_mod.Oracle(m).residual(z)
    nx = m.shape[0]
    scale = np.abs(r[:m.n_u]).max()
    corners = {0, nx, (nx + 1) * nx, (nx + 1) * (nx + 1) - 1}
    checked = 0
    for s, ms in zip(m.mpc_slave, m.mpc_master):
        if s // 2 in corners or ms // 2 in corners:
            continue
        assert abs(r[s] + r[ms]) < 1e-14 * scale * 10
        checked += 1
    assert checked > 20


# ---------------------------------------------------------------------------------- HVP

@pytest.mark.parametrize("dim", [2, 3])
def test_le_hvp_is_textbook_K_v(oracle_mod, dim):
    m = small_mesh(dim, 0)
    K = tb.stiffness(m)
    v = fi.random_direction(m.n_u, 5)
    y = oracle_mod.Oracle(m).hvp(fi.generic_state(m, 1), v)
    assert np.abs(y - K @ v).max() < 1e-14 * np.abs(K @ v).max() * 10


@pytest.mark.parametrize("dim", [2, 3])
def test_nh_hvp_matches_residual_fd(oracle_mod, dim):
    m = small_mesh(dim, 1)
    o = oracle_mod.Oracle(m)
    u = fi.generic_state(m, 6)
    h = 1e-5
    for j in np.random.default_rng(1).choice(m.n_u, 5, replace=False):
        e = np.zeros(m.n_u); e[j] = 1.0
        y = o.hvp(u, e)
        fd = (o.residual(u + h * e) - o.residual(u - h * e)) / (2 * h)
        assert np.abs(y - fd).max() < 1e-8 * max(1.0, np.abs(y).max())


@pytest.mark.parametrize("dim,material", [(2, 1), (3, 1), (3, 0)])
def test_hvp_symmetry(oracle_mod, dim, material):
    m = small_mesh(dim, material)
    o = oracle_mod.Oracle(m)
    u = fi.generic_state(m, 7)
    v, w = fi.random_direction(m.n_u, 1), fi.random_direction(m.n_u, 2)
    a, b = v @ o.hvp(u, w), w @ o.hvp(u, v)
    assert abs(a - b) < 1e-14 * max(abs(a), 1.0) * 10
    H = o.dense_hessian(u)
    assert np.abs(H - H.T).max() < 1e-14 * np.abs(H).max() * 10


@pytest.mark.parametrize("dim", [2, 3])
def test_nh_tangent_at_zero_equals_le(oracle_mod, dim):
    m = small_mesh(dim, 1)
    v = fi.random_direction(m.n_u, 3)
    y_nh = oracle_mod.Oracle(m).hvp(np.zeros(m.n_u), v)
    y_le = oracle_mod.Oracle(m.copy_with(material=0)).hvp(np.zeros(m.n_u), v)
    assert np.abs(y_nh - y_le).max() < 1e-15 * np.abs(y_le).max() * 10


@pytest.mark.parametrize("dim,nullity", [(2, 3), (3, 6)])
def test_le_null_space_dimension(oracle_mod, dim, nullity):
    m = small_mesh(dim, 0)
    H = oracle_mod.Oracle(m).dense_hessian(np.zeros(m.n_u))
    ev = np.linalg.eigvalsh(H)
    assert np.sum(np.abs(ev) < 1e-10 * ev.max()) == nullity


@pytest.mark.parametrize("dim", [2, 3])
def test_tangent_patch_test(oracle_mod, dim):
    m = small_mesh(dim, 1)
    F = np.diag([1.1] + [0.95904] * (dim - 1))
    u = fi.affine_field(m, F - np.eye(dim))
    v = fi.affine_field(m, np.random.default_rng(4).uniform(-1, 1, (dim, dim)))
    y = oracle_mod.Oracle(m).hvp(u, v).reshape(-1, dim)
    interior = ~fi.boundary_node_mask(m)
    assert np.abs(y[interior]).max() < 1e-14 * np.abs(y).max() * 10


def test_hvp_bc_is_masked_operator(oracle_mod):
    m = fi.roller_bc(small_mesh(2, 1), 0.1)
    o = oracle_mod.Oracle(m)
    u = fi.lift(m, fi.generic_state(m, 8))
    v = fi.random_direction(m.n_u, 9)
    H = o.dense_hessian(u)
    Pf = np.ones(m.n_u); Pf[m.dirichlet_dofs] = 0.0
    ref = Pf * (H @ (Pf * v)) + (1 - Pf) * v
    assert np.abs(o.hvp(u, v, bc=True) - ref).max() < 1e-14 * np.abs(ref).max() * 10


def test_lagrangian_hessian_blocks(oracle_mod):
    # [[K, B^T], [B, 0]] (App. B)
    m = fi.config_mesh(5, n=5)
    o = oracle_mod.Oracle(m)
    z = fi.generic_state(m, 1)
    H = o.dense_hessian(z)
    K = tb.stiffness(m)
    B = tb.constraint_matrix(m)
    nu = m.n_u
    assert np.abs(H[:nu, :nu] - K).max() < 1e-13 * np.abs(K).max()
    assert np.array_equal(H[nu:, :nu], B)
    assert np.array_equal(H[:nu, nu:], B.T)
    assert np.all(H[nu:, nu:] == 0.0)
    assert np.linalg.matrix_rank(B) == m.n_mpc == 2 * (2 * 5 + 1)   # C13: full row rank


@pytest.mark.parametrize("material", [0, 1])
def test_patch_tests_on_unstructured_tets(oracle_mod, material):
    """Residual and tangent patch tests (§8(c3)) on the Delaunay Tet4 mesh (slivers, node
    degrees 13-30): exact on any P1 mesh, so the interior entries vanish to rounding."""
    m = fi.delaunay_tet4(300, 4, 11).copy_with(material=material)
    o = oracle_mod.Oracle(m)
    interior = ~fi.boundary_node_mask(m)
    A = np.random.default_rng(9).uniform(-0.08, 0.08, (3, 3))
    r = o.residual(fi.affine_field(m, A)).reshape(-1, 3)
    assert np.abs(r[interior]).max() < 1e-13 * np.abs(r).max()
    F = np.diag([1.1, 0.97, 0.97])
    v = fi.affine_field(m, np.random.default_rng(4).uniform(-1, 1, (3, 3)))
    y = o.hvp(fi.affine_field(m, F - np.eye(3)), v).reshape(-1, 3)
    assert np.abs(y[interior]).max() < 1e-13 * np.abs(y).max()
