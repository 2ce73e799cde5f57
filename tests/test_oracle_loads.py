"""Pins for the oracle's external loads (§6.1):
the traction and body-force nodal loads, checked against the SPEC worked examples, force
balance and the closed-form homogeneous solution of the uniaxial traction problem."""
import json
import os

import numpy as np
import pytest

import fem_inputs as fi

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def uniaxial_strain(lam, mu, t, dim):
    """Homogeneous linear-elastic strain under sigma_xx = t, other stresses free (3D) /
    plane strain eps_zz = 0 (2D): textbook Hooke's law with E, nu from (lambda, mu)."""
    E = mu * (3 * lam + 2 * mu) / (lam + mu)
    nu = lam / (2 * (lam + mu))
    if dim == 3:
        return np.diag([t / E, -nu * t / E, -nu * t / E])
    return np.diag([(1 - nu ** 2) * t / E, -nu * (1 + nu) * t / E])


def test_line2_equal_nodal_loads(oracle_mod):
    g = GOLD["traction_line2_equal_loads"]
    m = fi.Mesh(dim=2, coords=np.array(g["coords"]), conn=np.zeros((0, 3), np.int32))
    f = oracle_mod.Oracle(m).traction_load(np.array([g["facet"]]), np.array(g["t"]))
    assert np.abs(f.reshape(2, 2) - np.array(g["f"])).max() < 1e-15


@pytest.mark.parametrize("dim", [2, 3])
def test_traction_potential_of_constant_u(oracle_mod, dim):
    # constant u = c, constant t on a surface of measure A -> -A (t . c)
    base = fi.perturb(fi.grid_tri3(5, 5) if dim == 2 else fi.grid_tet4(3, 3, 3), 0.2, 2)
    fac = fi.boundary_facets(base, 0, 1.0)
    t = np.array([2.0, 1.0, -0.5])[:dim]
    c = np.array([0.3, -0.1, 0.2])[:dim]
    f = oracle_mod.Oracle(base).traction_load(fac, t)
    u = np.tile(c, base.n_nodes)
    assert abs(-(f @ u) - (-1.0 * t @ c)) < 1e-15   # the face x = 1 has measure 1


def test_body_force_balance(oracle_mod):
    m = fi.perturb(fi.grid_tet4(3, 3, 3), 0.2, 4)
    b = np.array([0.5, -1.0, 2.0])
    f = oracle_mod.Oracle(m).body_load(b).reshape(-1, 3)
    assert np.abs(f.sum(axis=0) - b).max() < 1e-15   # |Omega| = 1


@pytest.mark.parametrize("dim", [2, 3])
def test_uniaxial_traction_homogeneous_solution(oracle_mod, dim):
    # symmetry rollers on x=0, y=0 (, z=0), traction t on x = 1: the FE solution of the
    # linear-elastic problem is the homogeneous uniaxial field u = eps X on any P1 mesh
    base = fi.perturb(fi.grid_tri3(6, 6) if dim == 2 else fi.grid_tet4(3, 3, 3), 0.2, 5)
    m = fi.roller_symmetry_bc(base.copy_with(material=0))
    t = 0.02
    tv = np.zeros(dim)
    tv[0] = t
    f = oracle_mod.Oracle(m).traction_load(fi.boundary_facets(m, 0, 1.0), tv)
    mf = m.copy_with(f_ext=f)
    z, info = oracle_mod.Oracle(mf).newton(fi.lift(mf), atol=1e-14, rtol=1e-14, cg_rtol=1e-14)
    ref = fi.affine_field(m, uniaxial_strain(m.lam, m.mu, t, dim))
    assert np.abs(z - ref).max() <= 1e-12 * np.abs(ref).max()
