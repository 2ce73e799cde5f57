"""GPU parity for SURVEY §8(f) f3 (§6.1): traction / body-force loads
through the C ABI (fem_add_traction, fem_add_body_force) against the oracle's Gauss-rule
loads, and the traction problem solved by Newton against the oracle and the closed form."""
import numpy as np
import pytest

import fem_inputs as fi
from tests.test_oracle_loads import uniaxial_strain

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


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("dim", [2, 3])
def test_load_vectors(fem, oracle_mod, dim):
    base = fi.perturb(fi.grid_tri3(24, 24) if dim == 2 else fi.grid_tet4(7, 6, 5), 0.2, 3)
    rng = np.random.default_rng(1)
    fac = np.concatenate([fi.boundary_facets(base, 0, 1.0), fi.boundary_facets(base, 1, 0.0)])
    t = rng.uniform(-1, 1, size=(len(fac), dim))
    b = np.array([0.3, -0.7, 1.1])[:dim]
    prob = fem.Problem(base)
    prob.add_traction(fac, t)
    prob.add_body_force(b)
    o = oracle_mod.Oracle(base)
    ref = o.traction_load(fac, t) + o.body_load(b)
    assert rel(prob.f_ext(), ref) <= 1e-13


def test_traction_enters_energy_and_residual(fem, oracle_mod):
    base = fi.roller_symmetry_bc(fi.perturb(fi.grid_tet4(6, 5, 4), 0.1, 4))
    fac = fi.boundary_facets(base, 0, 1.0)
    o = oracle_mod.Oracle(base)
    f = o.traction_load(fac, np.array([0.05, 0.01, -0.02]))
    mf = base.copy_with(f_ext=f)
    z = fi.lift(mf, fi.generic_state(mf, 2))
    prob = fem.Problem(base)
    prob.add_traction(fac, [0.05, 0.01, -0.02])
    of = oracle_mod.Oracle(mf)
    assert abs(prob.energy(dev(z)).item() - of.energy(z)) <= 1e-12 * abs(of.energy(z))
    assert rel(prob.residual(dev(z), bc=True), of.residual(z, bc=True)) <= 1e-12


@pytest.mark.parametrize("dim", [2, 3])
def test_uniaxial_traction_newton(fem, dim):
    # LE: closed-form homogeneous solution on a perturbed mesh; one Newton step
    base = fi.perturb(fi.grid_tri3(40, 40) if dim == 2 else fi.grid_tet4(10, 9, 8), 0.1, 5)
    m = fi.roller_symmetry_bc(base.copy_with(material=0))
    tv = np.zeros(dim)
    tv[0] = 0.02
    prob = fem.Problem(m)
    prob.add_traction(fi.boundary_facets(m, 0, 1.0), tv)
    z, info = prob.newton_solve(dev(fi.lift(m)), atol=1e-14, rtol=1e-13, cg_rtol=1e-14)
    assert info["converged"] and info["iters"] <= 2
    ref = fi.affine_field(m, uniaxial_strain(m.lam, m.mu, 0.02, dim))
    assert rel(z, ref) <= 1e-10


def test_neo_hookean_traction_newton_matches_oracle(fem, oracle_mod):
    base = fi.roller_symmetry_bc(fi.perturb(fi.grid_tet4(5, 4, 4), 0.1, 6))
    fac = fi.boundary_facets(base, 0, 1.0)
    tv = np.array([0.08, 0.0, 0.0])
    f = oracle_mod.Oracle(base).traction_load(fac, tv)
    mf = base.copy_with(f_ext=f)
    ref, rinfo = oracle_mod.Oracle(mf).newton(fi.lift(mf), atol=1e-13, rtol=1e-12, cg_rtol=1e-13)
    prob = fem.Problem(base)
    prob.add_traction(fac, tv)
    z, info = prob.newton_solve(dev(fi.lift(base)), atol=1e-13, rtol=1e-12, cg_rtol=1e-13)
    assert info["converged"] and rinfo["status"] == 0
    assert rel(z, ref) <= 1e-10
