"""GPU parity for SURVEY §8(f) f4 (§3.1): the virtual-work
residual and non-symmetric JVP of the scalar advection-diffusion problem through the C ABI
(fem_vw_*) against the oracle's dual-number derivatives, and GMRES against dense solves."""
import numpy as np
import pytest

import fem_inputs as fi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fem():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_12365_b200 import build, fem as f
    build.build()
    return f


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def problem(dim, n, seed, D=0.05, m=0.0, bc=True):
    base = fi.perturb(fi.grid_tri3(n, n) if dim == 2 else fi.grid_tet4(n, n, n), 0.2, seed)
    X = base.coords
    # rigid rotation about the cell centre (divergence-free) plus a drift
    vel = np.zeros_like(X)
    vel[:, 0] = -(X[:, 1] - 0.5) + 0.2
    vel[:, 1] = (X[:, 0] - 0.5)
    dn = dv = None
    if bc:
        dn = np.nonzero(np.abs(X[:, 0]) < 1e-12)[0].astype(np.int32)
        dv = np.exp(-10 * (X[dn, 1] - 0.5) ** 2)
    return base, vel, dict(diffusivity=D, velocity=vel, mass_coef=m, dirichlet_nodes=dn,
                           dirichlet_vals=dv)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("bc", [False, True])
def test_residual_and_jvp_parity(fem, oracle_mod, dim, bc):
    base, vel, kw = problem(dim, 20 if dim == 2 else 6, 3, m=2.0)
    rng = np.random.default_rng(4)
    c, cold, x = rng.uniform(-1, 1, (3, base.n_nodes))
    g = fem.VirtualWorkProblem(base.coords, base.conn, **kw)
    o = oracle_mod.VwOracle(base.coords, base.conn, **kw)
    assert rel(g.residual(c, cold, bc=bc), o.residual(c, cold, bc=bc)) <= 1e-12
    assert rel(g.jvp(x, bc=bc), o.jvp(x, bc=bc)) <= 1e-12


def test_gmres_steady_solution_matches_dense_solve(fem, oracle_mod):
    base, vel, kw = problem(2, 16, 5)
    o = oracle_mod.VwOracle(base.coords, base.conn, **kw)
    c0 = np.zeros(base.n_nodes)
    c0[kw["dirichlet_nodes"]] = kw["dirichlet_vals"]
    ref = c0 + np.linalg.solve(o.dense(bc=True), -o.residual(c0, bc=True))
    g = fem.VirtualWorkProblem(base.coords, base.conn, **kw)
    ct = torch.zeros(base.n_nodes, dtype=torch.float64, device="cuda")
    g.apply_dirichlet(ct)
    b = -g.residual(ct, bc=True)
    dx, info = g.gmres_solve(b, restart=40, rtol=1e-13)
    assert info["converged"]
    assert rel(ct + dx, ref) <= 1e-10


def test_gmres_transient_steps_match_oracle(fem, oracle_mod):
    # backward-Euler steps (m = 1/dt, lumped mass) of the advected pulse: each step solves
    # K c = m V c_old with GMRES; compare 3 steps with dense solves
    base, vel, kw = problem(2, 12, 6, D=0.01, m=20.0, bc=False)
    X = base.coords
    c = np.exp(-40 * ((X[:, 0] - 0.3) ** 2 + (X[:, 1] - 0.5) ** 2))
    o = oracle_mod.VwOracle(base.coords, base.conn, **kw)
    K = o.dense()
    g = fem.VirtualWorkProblem(base.coords, base.conn, **kw)
    cg = torch.as_tensor(c, device="cuda")
    cr = c.copy()
    for _ in range(3):
        r0 = o.residual(np.zeros_like(cr), cr)          # = -m V c_old
        cr = np.linalg.solve(K, -r0)
        b = -g.residual(torch.zeros_like(cg), cg)
        cg, info = g.gmres_solve(b, x0=cg, restart=30, rtol=1e-13)
        assert info["converged"]
    assert rel(cg, cr) <= 1e-10


def test_vw_errors(fem):
    base, vel, kw = problem(2, 4, 7)
    bad = base.conn.copy()
    bad[0, 0] = base.n_nodes + 5
    with pytest.raises(fem.FemError):
        fem.VirtualWorkProblem(base.coords, bad, **kw)


def test_gmres_zero_rhs_and_restart_bounds(fem):
    base, vel, kw = problem(2, 4, 8)
    g = fem.VirtualWorkProblem(base.coords, base.conn, **kw)
    x, info = g.gmres_solve(torch.zeros(base.n_nodes, dtype=torch.float64, device="cuda"))
    assert info["converged"] and info["iters"] == 0
    with pytest.raises(fem.FemError):
        g.gmres_solve(torch.ones(base.n_nodes, dtype=torch.float64, device="cuda"), restart=0)
