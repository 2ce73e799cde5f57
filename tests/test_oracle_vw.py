"""Pins for the oracle's virtual-work path (§3.1, P:224-236;
advection-diffusion P:772-802): residual and JVP of the scalar advection-diffusion virtual
work, checked against closed forms, finite differences, symmetry / asymmetry witnesses and
the textbook 1D steady solution — not against the oracle itself."""
import numpy as np
import pytest

import fem_inputs as fi


def strip(n=40, ny=2, perturb=0.0, seed=1):
    m = fi.grid_tri3(n, ny)
    if perturb:
        m = fi.perturb(m, perturb, seed)
    return m


def lumped(m):
    X = m.coords[m.conn]
    vol = 0.5 * ((X[:, 1, 0] - X[:, 0, 0]) * (X[:, 2, 1] - X[:, 0, 1])
                 - (X[:, 2, 0] - X[:, 0, 0]) * (X[:, 1, 1] - X[:, 0, 1]))
    V = np.zeros(m.n_nodes)
    np.add.at(V, m.conn.ravel(), np.repeat(vol / 3, 3))
    return V


def test_constant_field_has_zero_residual(oracle_mod):
    m = strip(8, 8, 0.2)
    vel = np.random.default_rng(0).uniform(-1, 1, (m.n_nodes, 2))
    o = oracle_mod.VwOracle(m.coords, m.conn, 0.3, vel)
    assert np.abs(o.residual(np.full(m.n_nodes, 2.5))).max() < 1e-15
    assert np.abs(o.jvp(np.ones(m.n_nodes))).max() < 1e-14


def test_linear_field_residual_closed_form(oracle_mod):
    # c = g.X, uniform velocity w: the diffusion part vanishes at interior nodes (patch test)
    # and the advection part is (w . g) times the lumped nodal volume
    m = strip(8, 8, 0.2, 3)
    g, w = np.array([0.7, -0.4]), np.array([1.5, 0.5])
    o = oracle_mod.VwOracle(m.coords, m.conn, 0.2, np.tile(w, (m.n_nodes, 1)))
    r = o.residual(m.coords @ g)
    interior = ~fi.boundary_node_mask(m)
    ref = (w @ g) * lumped(m)
    assert np.abs(r[interior] - ref[interior]).max() < 1e-15


def test_zero_velocity_is_symmetric_and_advection_is_not(oracle_mod):
    m = strip(6, 6, 0.2, 4)
    K0 = oracle_mod.VwOracle(m.coords, m.conn, 0.5, np.zeros((m.n_nodes, 2))).dense()
    assert np.abs(K0 - K0.T).max() < 1e-14
    assert np.linalg.eigvalsh(0.5 * (K0 + K0.T)).min() > -1e-12        # diffusion: PSD
    vel = np.tile([1.0, 0.3], (m.n_nodes, 1))
    K = oracle_mod.VwOracle(m.coords, m.conn, 0.5, vel).dense()
    assert np.abs(K - K.T).max() > 1e-3                                  # asymmetry witness
    # the symmetric part of the advection operator is the boundary flux only: for a
    # constant velocity, 1^T K_adv c = sum_e vol (w . grad c) = boundary integral
    assert np.abs((K - K0).sum(axis=0)).max() > 0


def test_jvp_matches_finite_differences_of_residual(oracle_mod):
    m = strip(5, 5, 0.2, 5)
    rng = np.random.default_rng(2)
    vel = rng.uniform(-1, 1, (m.n_nodes, 2))
    o = oracle_mod.VwOracle(m.coords, m.conn, 0.1, vel, mass_coef=3.0)
    c, x, cold = rng.uniform(-1, 1, (3, m.n_nodes))
    h = 1e-6
    fd = (o.residual(c + h * x, cold) - o.residual(c - h * x, cold)) / (2 * h)
    assert np.abs(o.jvp(x) - fd).max() < 1e-8


def test_steady_1d_profile_converges(oracle_mod):
    # -D c'' + w c' = 0 on [0, 1], c(0) = 1, c(1) = 0 on a strip: the FE solution approaches
    # c(x) = (e^{Pe} - e^{Pe x}) / (e^{Pe} - 1), Pe = w / D (first order in h on the
    # diagonal-split strip: the error halves with h; a wrong advection sign or scale does not
    # converge)
    errs = []
    for n in (20, 40):
        m = strip(n, 1)
        D, w = 0.25, 1.0
        left = np.nonzero(np.abs(m.coords[:, 0]) < 1e-12)[0]
        right = np.nonzero(np.abs(m.coords[:, 0] - 1) < 1e-12)[0]
        dn = np.concatenate([left, right]).astype(np.int32)
        dv = np.concatenate([np.ones(len(left)), np.zeros(len(right))])
        o = oracle_mod.VwOracle(m.coords, m.conn, D, np.tile([w, 0.0], (m.n_nodes, 1)),
                                dirichlet_nodes=dn, dirichlet_vals=dv)
        c0 = np.zeros(m.n_nodes)
        c0[dn] = dv
        K = o.dense(bc=True)
        c = c0 + np.linalg.solve(K, -o.residual(c0, bc=True))
        Pe = w / D
        exact = (np.exp(Pe) - np.exp(Pe * m.coords[:, 0])) / (np.exp(Pe) - 1)
        errs.append(np.abs(c - exact).max())
    assert errs[1] < errs[0] / 1.8 and errs[1] < 6e-3
