"""Pins for the oracle's f2 pieces (§6.2.2): the
volume-averaged stress (fem_ref_mean_stress) and the stationary point of the periodic
Lagrangian by dense Newton (Oracle.newton_dense), checked against closed forms and the
textbook Hill bounds, never against the oracle itself.
"""
import numpy as np
import pytest

import fem_inputs as fi

LAM, MU = 0.57692307692307687, 0.38461538461538458       # E = 1, nu = 0.3 (reading C3)
PHASES = ((LAM, MU), (10 * LAM, 10 * MU))                  # matrix, 10x stiffer inclusion


def c_iso(lam, mu, dim=2):
    """Isotropic stiffness in Voigt notation with engineering shear (plane strain in 2D)."""
    if dim == 2:
        return np.array([[lam + 2 * mu, lam, 0.0], [lam, lam + 2 * mu, 0.0], [0.0, 0.0, mu]])
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    C[np.arange(3), np.arange(3)] = lam + 2 * mu
    C[np.arange(3, 6), np.arange(3, 6)] = mu
    return C


def textbook_P(A, lam, mu, material):
    """First Piola-Kirchhoff stress from the textbook closed forms (not the oracle's dual
    numbers): LE sigma = 2 mu eps + lam tr(eps) I; NH P = mu (F - F^-T) + lam ln J F^-T."""
    d = A.shape[0]
    if material == 0:
        eps = 0.5 * (A + A.T)
        return 2 * mu * eps + lam * np.trace(eps) * np.eye(d)
    F = np.eye(d) + A
    FiT = np.linalg.inv(F).T
    return mu * (F - FiT) + lam * np.log(np.linalg.det(F)) * FiT


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("material", [0, 1])
def test_mean_stress_affine_closed_form(oracle_mod, dim, material):
    # u = A X on a perturbed mesh: every element has H = A, so <P> = P(A) exactly and
    # |Omega| = 1 (P1 patch property)
    base = fi.grid_tri3(6, 6) if dim == 2 else fi.grid_tet4(3, 3, 3)
    m = fi.perturb(base, 0.2, 3).copy_with(material=material)
    A = np.array([[0.03, -0.01, 0.02], [0.015, -0.02, 0.01], [0.0, 0.01, 0.025]])[:dim, :dim]
    sig, vol = oracle_mod.Oracle(m).mean_stress(fi.affine_field(m, A))
    assert abs(vol - 1.0) < 1e-14
    ref = textbook_P(A, m.lam, m.mu, material)
    assert np.abs(sig - ref).max() <= 1e-14 * np.abs(ref).max()


def test_mean_stress_two_phase_is_volume_weighted(oracle_mod):
    # phase-wise constant strain A: <P> = f1 P_1(A) + f2 P_2(A) with the phase volume fractions
    m = fi.two_phase(fi.perturb(fi.grid_tri3(8, 8), 0.2, 4).copy_with(material=0), 0.3, *PHASES)
    A = np.array([[0.01, 0.004], [0.002, -0.006]])
    sig, _ = oracle_mod.Oracle(m).mean_stress(fi.affine_field(m, A))
    X = m.coords[m.conn]
    vol = 0.5 * np.abs((X[:, 1, 0] - X[:, 0, 0]) * (X[:, 2, 1] - X[:, 0, 1])
                       - (X[:, 2, 0] - X[:, 0, 0]) * (X[:, 1, 1] - X[:, 0, 1]))
    f1 = vol[m.phase == 1].sum() / vol.sum()
    ref = (1 - f1) * textbook_P(A, *PHASES[0], 0) + f1 * textbook_P(A, *PHASES[1], 0)
    assert 0.1 < f1 < 0.5
    assert np.abs(sig - ref).max() <= 1e-14 * np.abs(ref).max()


PAIRS2 = [(0, 0), (1, 1), (0, 1)]        # Voigt order, engineering shear


def unit_strain(i, j):
    e = np.zeros((2, 2))
    e[i, j] += 0.5
    e[j, i] += 0.5
    return e


def oracle_c_hom(oracle_mod, base):
    cols = []
    for e in (unit_strain(i, j) for i, j in PAIRS2):
        m = fi.periodic_mpc(base, e)
        o = oracle_mod.Oracle(m)
        z, info = o.newton_dense(fi.lift(m), atol=1e-13, rtol=1e-13)
        assert info["converged"] and info["iters"] <= 2     # linear: one step
        g = m.mpc_offset
        u = z[:m.n_u]
        assert np.abs(u[m.mpc_slave] - u[m.mpc_master] - g).max() < 1e-13   # g(u) = 0
        sig = o.mean_stress(z)[0]
        cols.append(np.array([0.5 * (sig[i, j] + sig[j, i]) for i, j in PAIRS2]))
    return np.stack(cols, axis=1)


def test_homogeneous_rve_gives_the_material_stiffness(oracle_mod):
    # u = eps_hat X solves the periodic problem of a homogeneous cell exactly => C_hom = C
    base = fi.perturb(fi.grid_tri3(8, 8), 0.2, 5).copy_with(material=0)
    C = oracle_c_hom(oracle_mod, base)
    ref = c_iso(base.lam, base.mu)
    assert np.abs(C - ref).max() <= 1e-12 * np.abs(ref).max()


def test_two_phase_rve_within_hill_bounds(oracle_mod):
    # textbook bounds: Reuss (harmonic) <= C_hom <= Voigt (arithmetic mean) as quadratic
    # forms; the conforming FE solution is stiffer than the exact one, so the Voigt bound
    # (affine trial field) is strict and the Reuss bound holds a fortiori; C_hom symmetric
    # (discrete Hill-Mandel: <P> : e = 2 W / |Omega| at equilibrium)
    base = fi.two_phase(fi.perturb(fi.grid_tri3(10, 10), 0.1, 6).copy_with(material=0), 0.3, *PHASES)
    C = oracle_c_hom(oracle_mod, base)
    X = base.coords[base.conn]
    vol = 0.5 * np.abs((X[:, 1, 0] - X[:, 0, 0]) * (X[:, 2, 1] - X[:, 0, 1])
                       - (X[:, 2, 0] - X[:, 0, 0]) * (X[:, 1, 1] - X[:, 0, 1]))
    f1 = vol[base.phase == 1].sum() / vol.sum()
    C0, C1 = c_iso(*PHASES[0]), c_iso(*PHASES[1])
    CV = (1 - f1) * C0 + f1 * C1
    CR = np.linalg.inv((1 - f1) * np.linalg.inv(C0) + f1 * np.linalg.inv(C1))
    assert np.abs(C - C.T).max() <= 1e-10 * np.abs(C).max()
    assert np.linalg.eigvalsh(0.5 * (CV - C + (CV - C).T)).min() > 0
    assert np.linalg.eigvalsh(0.5 * (C - CR + (C - CR).T)).min() > 0
