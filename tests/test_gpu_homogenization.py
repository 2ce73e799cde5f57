"""GPU parity for SURVEY §8(f) f2 (§6.2.2): MINRES on the periodic
Lagrangian's saddle-point operator, Newton-MINRES, the volume-averaged stress and the
homogenized stiffness, through the C ABI, against the oracle's dense Newton and closed forms.
"""
import numpy as np
import pytest

import fem_inputs as fi
from tests.test_oracle_homogenization import PHASES, c_iso, oracle_c_hom

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


def rve(n=12, material=0):
    base = fi.two_phase(fi.perturb(fi.grid_tri3(n, n), 0.1, 7).copy_with(material=material), 0.3,
                        *PHASES)
    return fi.periodic_mpc(base, np.array([[0.01, 0.005], [0.005, -0.003]]))


def test_minres_saddle_point_matches_dense_solve(fem, oracle_mod):
    m = rve()
    o = oracle_mod.Oracle(m)
    z0 = fi.lift(m)
    b = -o.residual(z0, bc=True)
    ref = np.linalg.solve(o.dense_hessian(z0, bc=True), b)
    prob = fem.Problem(m)
    x, info = prob.minres_solve(dev(b), z=dev(z0), rtol=1e-14, max_iter=20000)
    assert info["converged"]
    assert rel(x, ref) <= 1e-10
    assert info["res"] <= 1e-12 * np.linalg.norm(b)


def test_minres_csr_operator(fem, oracle_mod):
    m = rve(10)
    o = oracle_mod.Oracle(m)
    z0 = fi.lift(m)
    b = -o.residual(z0, bc=True)
    ref = np.linalg.solve(o.dense_hessian(z0, bc=True), b)
    prob = fem.Problem(m)
    vals = prob.assemble_csr(dev(z0), bc=True)
    x, info = prob.minres_solve(dev(b), vals=vals, op=1, rtol=1e-14, max_iter=20000, check_every=8)
    assert info["converged"] and rel(x, ref) <= 1e-10


def test_minres_on_spd_system_equals_cg(fem):
    m = fi.roller_bc(fi.perturb(fi.grid_tri3(16, 16), 0.2, 9).copy_with(material=1), 0.05)
    z = dev(fi.lift(m, fi.generic_state(m, 1)))
    b = fi.random_direction(m.n_total, 2)
    b[m.dirichlet_dofs] = 0.0
    prob = fem.Problem(m)
    xc, _ = prob.cg_solve(dev(b), z=z, rtol=1e-14)
    xm, info = prob.minres_solve(dev(b), z=z, rtol=1e-14)
    assert info["converged"] and rel(xm, xc.cpu().numpy()) <= 1e-10


@pytest.mark.parametrize("material", [0, 1])
def test_newton_minres_periodic_matches_dense_newton(fem, oracle_mod, material):
    # LE: one step; NH: nonlinear periodic Lagrangian, quadratic convergence
    m = rve(10, material)
    ref, rinfo = oracle_mod.Oracle(m).newton_dense(fi.lift(m), atol=1e-13, rtol=1e-12)
    assert rinfo["converged"]
    prob = fem.Problem(m)
    z, info = prob.newton_solve(dev(fi.lift(m)), atol=1e-13, rtol=1e-12, cg_rtol=1e-13,
                                check_every=8)
    assert info["converged"]
    assert rel(z[:m.n_u], ref[:m.n_u]) <= 1e-10
    u = z[:m.n_u].cpu().numpy()
    assert np.abs(u[m.mpc_slave] - u[m.mpc_master] - m.mpc_offset).max() < 1e-10


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("material", [0, 1])
def test_mean_stress_parity(fem, oracle_mod, dim, material):
    base = fi.grid_tri3(20, 20) if dim == 2 else fi.grid_tet4(6, 6, 6)
    m = fi.two_phase(fi.perturb(base, 0.2, 10).copy_with(material=material), 0.3, *PHASES)
    z = fi.lift(m, fi.generic_state(m, 3))
    sig, vol = fem.Problem(m).mean_stress(dev(z))
    rsig, rvol = oracle_mod.Oracle(m).mean_stress(z)
    assert abs(vol - rvol) <= 1e-14
    assert np.abs(sig - rsig).max() <= 1e-12 * np.abs(rsig).max()


def test_homogenized_stiffness(fem, oracle_mod):
    from paper_2602_12365_b200.homogenize import homogenized_stiffness
    base = fi.two_phase(fi.perturb(fi.grid_tri3(10, 10), 0.1, 6).copy_with(material=0), 0.3,
                        *PHASES)
    C, reps = homogenized_stiffness(lambda e: fi.periodic_mpc(base, e), 2)
    ref = oracle_c_hom(oracle_mod, base)
    assert np.abs(C - ref).max() <= 1e-10 * np.abs(ref).max()
    hom = fi.perturb(fi.grid_tri3(10, 10), 0.1, 6).copy_with(material=0)
    C0, _ = homogenized_stiffness(lambda e: fi.periodic_mpc(hom, e), 2)
    ref0 = c_iso(hom.lam, hom.mu)
    assert np.abs(C0 - ref0).max() <= 1e-10 * np.abs(ref0).max()


def test_minres_zero_rhs_and_iteration_cap(fem):
    m = rve(6)
    prob = fem.Problem(m)
    z0 = dev(fi.lift(m))
    x, info = prob.minres_solve(torch.zeros(m.n_total, dtype=torch.float64, device="cuda"), z=z0)
    assert info["converged"] and info["iters"] == 0 and float(x.abs().max()) == 0.0
    b = dev(fi.random_direction(m.n_total, 3))
    _, info = prob.minres_solve(b, z=z0, rtol=1e-30, max_iter=5, raise_on_fail=False)
    assert info["status"] == 6 and info["iters"] == 5        # FEM_ERR_NOT_CONVERGED


def test_minres_graph_batches_match_direct_launches(fem, monkeypatch):
    # MINRES iterations between host checks replay a 3-iteration CUDA graph (the buffer
    # rotation has period 3); with the deterministic CSR operator the iterates are identical
    m = rve(12)
    prob = fem.Problem(m)
    z0 = dev(fi.lift(m))
    vals = prob.assemble_csr(z0, bc=True)
    b = dev(fi.random_direction(m.n_total, 4))
    xg, ig = prob.minres_solve(b, vals=vals, op=1, rtol=1e-13, check_every=9)
    monkeypatch.setenv("FEM_NO_GRAPHS", "1")
    xd, idd = prob.minres_solve(b, vals=vals, op=1, rtol=1e-13, check_every=9)
    assert ig["converged"] and idd["converged"] and ig["iters"] == idd["iters"]
    assert torch.equal(xg, xd)
