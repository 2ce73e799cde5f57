"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Floating point: normwise relative error <= 1e-12 (north_star; reading C14).
Pattern and coloring: bit-exact.  Converged Newton displacements: <= 1e-10 relative.
Small meshes span several 256-thread tiles plus a ragged tail; full BASELINE sizes are
checked on sampled rows the oracle computes one by one, and by size-independent
properties (patch tests, closed-form homogeneous solutions).
"""
import numpy as np
import pytest

import fem_inputs as fi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def fem():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_12365_b200 import build, fem as f
    build.build()
    return f


def rel(a, b):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def dev(x):
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda")


def meshes():
    out = {
        "cfg1-2d-le": fi.config_mesh(1),
        "2d-nh-roller": fi.roller_bc(fi.perturb(fi.grid_tri3(23, 17), 0.2, 3).copy_with(material=1), 0.1),
        "2d-nh-clamped": fi.clamped_bc(fi.perturb(fi.grid_tri3(19, 20), 0.2, 4).copy_with(material=1), 0.05),
        "3d-le": fi.roller_bc(fi.perturb(fi.grid_tet4(7, 6, 5), 0.1, 5).copy_with(material=0), 0.05),
        "3d-nh": fi.roller_bc(fi.perturb(fi.grid_tet4(6, 7, 5), 0.1, 6).copy_with(material=1), 0.05),
        "2d-le-mpc": fi.config_mesh(5, n=13),
        "3d-nh-shuffled": fi.renumber_nodes(fi.grid_tet4(5, 4, 6).copy_with(material=1), 21),
        "2d-nh-delaunay": fi.roller_bc(fi.delaunay_tri3(1800, 30, 7).copy_with(material=1), 0.05),
        # unstructured tets (App. A): node degrees 13-30, > 16 slots on many nodes
        "3d-nh-delaunay": fi.roller_bc(fi.delaunay_tet4(1500, 6, 7).copy_with(material=1), 0.05),
        # coarse surface grid around dense interior points: surface nodes with up to 80 incident
        # tets and 45 neighbours (beyond the node-tile and row-plan caps: the row-gather
        # fallback at high degree)
        "3d-nh-delaunay-graded": fi.roller_bc(fi.delaunay_tet4(3000, 3, 7).copy_with(material=1), 0.05),
    }
    ph = fi.two_phase(fi.perturb(fi.grid_tri3(16, 16), 0.2, 8).copy_with(material=1), 0.3,
                      (0.5, 0.3), (5.0, 3.0))
    ph = ph.copy_with(f_ext=np.random.default_rng(3).uniform(-1e-3, 1e-3, ph.n_u))
    out["2d-nh-phases-fext"] = ph
    return out


MESHES = meshes()
# state noise (x h) per mesh where the default 1e-2 inverts slivers (reading R11)
NOISE = {"3d-nh-delaunay-graded": 1e-4}


@pytest.fixture(scope="module", params=sorted(MESHES))
def case(request, fem, oracle_mod):
    mesh = MESHES[request.param]
    prob = fem.Problem(mesh)
    ref = oracle_mod.Oracle(mesh)
    z = fi.lift(mesh, fi.generic_state(mesh, 1, noise=NOISE.get(request.param, 0.01)))
    v = fi.random_direction(mesh.n_total, 2)
    return request.param, mesh, prob, ref, z, v


def test_energy(case):
    name, mesh, prob, ref, z, v = case
    e = prob.energy(dev(z)).item()
    r = ref.energy(z)
    assert abs(e - r) <= TOL * abs(r)


@pytest.mark.parametrize("bc", [False, True])
def test_residual(case, bc):
    name, mesh, prob, ref, z, v = case
    assert rel(prob.residual(dev(z), bc=bc), ref.residual(z, bc=bc)) <= TOL


@pytest.mark.parametrize("flag", [0, "DETERMINISTIC"])
def test_energy_residual_one_pass(case, fem, flag):
    """fem_energy_residual (value and gradient from one element pass) against the oracle."""
    name, mesh, prob, ref, z, v = case
    f = getattr(fem, flag) if flag else 0
    e, r = prob.energy_residual(dev(z), bc=True, flags=f)
    re = ref.energy(z)
    assert abs(e.item() - re) <= TOL * abs(re)
    assert rel(r, ref.residual(z, bc=True)) <= TOL


@pytest.mark.parametrize("bc", [False, True])
def test_hvp(case, bc):
    name, mesh, prob, ref, z, v = case
    assert rel(prob.hvp(dev(z), dev(v), bc=bc), ref.hvp(z, v, bc=bc)) <= TOL


@pytest.mark.parametrize("flag", ["DETERMINISTIC", "BASELINE_SCATTER", "STREAM_GEOM", "REFERENCE_METRIC", "COLORED_SCATTER",
                                  "TILE_COLORED"])
def test_residual_hvp_modes(case, fem, flag):
    name, mesh, prob, ref, z, v = case
    f = getattr(fem, flag)
    r1 = prob.residual(dev(z), bc=True, flags=f).cpu().numpy()
    y1 = prob.hvp(dev(z), dev(v), bc=True, flags=f).cpu().numpy()
    assert rel(r1, ref.residual(z, bc=True)) <= TOL
    assert rel(y1, ref.hvp(z, v, bc=True)) <= TOL
    if flag in ("DETERMINISTIC", "COLORED_SCATTER", "TILE_COLORED"):   # fixed summation orders
        assert np.array_equal(r1, prob.residual(dev(z), bc=True, flags=f).cpu().numpy())
        assert np.array_equal(y1, prob.hvp(dev(z), dev(v), bc=True, flags=f).cpu().numpy())


def test_pattern_bit_exact(case):
    name, mesh, prob, ref, z, v = case
    rp, ci = prob.sparsity()
    rrp, rci = ref.sparsity()
    assert np.array_equal(rp.cpu().numpy(), rrp)
    assert np.array_equal(ci.cpu().numpy(), rci)


def test_coloring_bit_exact(case):
    name, mesh, prob, ref, z, v = case
    colors, nc = prob.color()
    rcol, rnc = ref.colors()
    assert nc == rnc
    assert np.array_equal(colors.cpu().numpy(), rcol)


@pytest.mark.parametrize("mode", ["batched", "literal", "rows", "scatter", "colored"])
@pytest.mark.parametrize("bc", [False, True])
def test_assembly(case, mode, bc):
    name, mesh, prob, ref, z, v = case
    if mode == "colored" and mesh.n_mpc:
        pytest.skip("fused colored form: node-color seeds, no multiplier columns")
    vals = prob.assemble_csr(dev(z), bc=bc, mode=mode)
    assert rel(vals, ref.assemble_alg2(z, bc=bc)) <= TOL


def test_rows_mode_is_bitwise_reproducible(case):
    name, mesh, prob, ref, z, v = case
    a = prob.assemble_csr(dev(z), bc=True, mode="rows").cpu().numpy()
    b = prob.assemble_csr(dev(z), bc=True, mode="rows").cpu().numpy()
    assert np.array_equal(a, b)


def test_spmv_equals_hvp(case):
    name, mesh, prob, ref, z, v = case
    vals = prob.assemble_csr(dev(z), bc=True)
    y = prob.spmv(vals, dev(v))
    assert rel(y, ref.hvp(z, v, bc=True)) <= TOL
    rp, ci = ref.sparsity()
    import oracle
    assert rel(y, oracle.spmv(rp, ci, vals.cpu().numpy(), v)) <= TOL


def test_cg_matrix_free_and_csr(case):
    name, mesh, prob, ref, z, v = case
    if mesh.n_mpc:
        pytest.skip("saddle-point system: CG does not apply (SURVEY §8(f) f2)")
    b = v.copy()
    b[mesh.dirichlet_dofs] = 0.0
    if len(mesh.dirichlet_dofs) == 0:
        pytest.skip("singular without Dirichlet conditions")
    xr, rinfo = ref.cg(b, op=0, z=z, rtol=1e-13)
    x, info = prob.cg_solve(dev(b), z=dev(z), op=0, rtol=1e-13)
    assert info["converged"] and rinfo["status"] == 0
    assert rel(x, xr) <= 1e-10
    vals = prob.assemble_csr(dev(z), bc=True)
    x1, info1 = prob.cg_solve(dev(b), vals=vals, op=1, rtol=1e-13)
    assert info1["converged"] and rel(x1, xr) <= 1e-10
    x2, info2 = prob.cg_solve(dev(b), vals=vals, op=1, rtol=1e-13, jacobi=True)
    assert info2["converged"] and rel(x2, xr) <= 1e-10
    x3, info3 = prob.cg_solve(dev(b), vals=vals, op=1, rtol=1e-13, jacobi=2)   # node blocks
    assert info3["converged"] and rel(x3, xr) <= 1e-10


def test_newton(case):
    name, mesh, prob, ref, z, v = case
    if mesh.n_mpc or len(mesh.dirichlet_dofs) == 0 or mesh.f_ext is not None:
        pytest.skip("Newton parity on the roller / clamped problems")
    z0 = fi.lift(mesh)
    if "delaunay" in name:  # slivers next to x = L: start from the affine predictor (R2)
        z0 = fi.lift(mesh, fi.affine_field(mesh, np.diag([0.05] + [0.0] * (mesh.dim - 1))))
    zr, rinfo = ref.newton(z0, cg_rtol=1e-13)
    for op, jac in ((0, 0), (1, 0), (1, 2)):
        zg, info = prob.newton_solve(dev(z0), op=op, cg_rtol=1e-13, jacobi=jac)
        assert info["converged"] and rinfo["status"] == 0
        assert rel(zg, zr) <= 1e-10


@pytest.mark.parametrize("dim", [2, 3])
def test_newton_eisenstat_walker(fem, oracle_mod, dim):
    """Inexact Newton-Krylov (fem_newton_opts.forcing, reading R16): the same converged
    displacements as the oracle's exact-inner-solve Newton (<= 1e-10), with fewer CG
    iterations than fixed inner tolerances at the same outer target; MF and CSR operators."""
    if dim == 2:
        mesh = fi.config_mesh(2, n=40)
        eps = 0.1
    else:
        mesh = fi.config_mesh(3, n=10)
        eps = 0.05
    z0 = fi.lift(mesh, fi.affine_field(mesh, np.diag([eps] + [0.0] * (dim - 1))))
    zr, rinfo = oracle_mod.Oracle(mesh).newton(z0, cg_rtol=1e-13)
    assert rinfo["status"] == 0
    prob = fem.Problem(mesh)
    kw = dict(cg_rtol=1e-13, rtol=1e-12, atol=1e-16)
    zf, info_f = prob.newton_solve(dev(z0), op=0, **kw)
    for op, jac in ((0, 0), (1, 2)):
        ze, info_e = prob.newton_solve(dev(z0), op=op, jacobi=jac, forcing=0.9, **kw)
        assert info_e["converged"] and info_e["res"] <= 1e-12 * info_e["res0"]
        assert rel(ze, zr) <= 1e-10
    ze, info_e = prob.newton_solve(dev(z0), op=0, forcing=0.9, **kw)
    assert info_f["converged"] and info_e["cg_iters"] < info_f["cg_iters"]
    for bad in (-0.5, 1.5):
        with pytest.raises(RuntimeError):
            prob.newton_solve(dev(z0), op=0, forcing=bad, **kw)


# ------------------------------------------------------------------ edge cases

def test_single_element_and_empty(fem, oracle_mod):
    tri = fi.Mesh(dim=2, coords=np.array([[0., 0.], [1., 0.], [0., 1.]]),
                  conn=np.array([[0, 1, 2]], np.int32), material=1)
    p = fem.Problem(tri)
    z = np.array([0.01, 0.0, 0.02, -0.01, 0.0, 0.03])
    v = np.arange(6.0)
    o = oracle_mod.Oracle(tri)
    assert rel(p.hvp(dev(z), dev(v)), o.hvp(z, v)) <= TOL
    assert p.color()[1] == 6
    empty = fi.Mesh(dim=3, coords=np.zeros((4, 3)), conn=np.zeros((0, 4), np.int32))
    pe = fem.Problem(empty)
    assert pe.energy(torch.zeros(12, dtype=torch.float64, device="cuda")).item() == 0.0
    assert pe.nnz() == 0


def test_errors(fem):
    deg = fi.Mesh(dim=2, coords=np.array([[0., 0.], [1., 0.], [2., 0.]]),
                  conn=np.array([[0, 1, 2]], np.int32))
    with pytest.raises(fem.FemError) as ei:
        fem.Problem(deg)
    assert ei.value.status == 2
    bad = fi.Mesh(dim=2, coords=np.array([[0., 0.], [1., 0.], [0., 1.]]),
                  conn=np.array([[0, 1, 5]], np.int32))
    with pytest.raises(fem.FemError) as ei:
        fem.Problem(bad)
    assert ei.value.status == 1
    tri = fi.Mesh(dim=2, coords=np.array([[0., 0.], [1., 0.], [0., 1.]]),
                  conn=np.array([[0, 1, 2]], np.int32), material=1)
    p = fem.Problem(tri)
    z = dev(np.array([0.0, 0.0, -3.0, 0.0, 0.0, 0.0]))   # folds the element: J < 0
    p.residual(z)
    with pytest.raises(fem.FemError) as ei:
        p.check()
    assert ei.value.status == 3
    with pytest.raises(ValueError):
        p.hvp(z, dev(np.zeros(5)))


@pytest.mark.parametrize("dim", [2, 3])
def test_inverted_element_every_op(fem, dim):
    """J <= 0 (InvertedElement) is reported by every NH kernel: energy,
    residual (both forms), the one-pass energy+residual, HVP (tile, deterministic, baseline
    scatter), linearize and the assembly (every mode)."""
    mesh = fi.grid_tri3(3, 3) if dim == 2 else fi.grid_tet4(3, 3, 3)
    mesh = mesh.copy_with(material=fi.NEO_HOOKEAN)
    p = fem.Problem(mesh)
    z = np.zeros(mesh.n_total)
    z[0:dim] = 5.0   # corner node 0 pushed through the opposite faces of its elements: J < 0
    zt, vt = dev(z), dev(np.ones(mesh.n_total))
    calls = [lambda: p.energy(zt), lambda: p.residual(zt), lambda: p.energy_residual(zt),
             lambda: p.hvp(zt, vt), lambda: p.hvp(zt, vt, flags=fem.DETERMINISTIC),
             lambda: p.hvp(zt, vt, flags=fem.BASELINE_SCATTER), lambda: p.linearize(zt),
             lambda: p.residual(zt, flags=fem.BASELINE_SCATTER)]
    calls += [lambda m=m: p.assemble_csr(zt, mode=m) for m in ("rows", "batched", "scatter")]
    for call in calls:
        with pytest.raises(fem.FemError) as ei:
            call()
            p.check()
        assert ei.value.status == 3
    p.check()   # the error word is cleared once reported


# ------------------------------------------------------------------ full BASELINE sizes

def sampled_rows(n, k, seed):
    rows = np.random.default_rng(seed).choice(n, k, replace=False)
    return np.unique(np.concatenate([rows, [0, n - 1]]))


@pytest.mark.parametrize("cfg", [2, 3])
def test_full_size_sampled_parity(fem, oracle_mod, cfg):
    mesh = fi.config_mesh(cfg)
    prob = fem.Problem(mesh)
    ref = oracle_mod.Oracle(mesh)
    h = mesh.length / max(mesh.shape)
    z = fi.lift(mesh, fi.generic_state(mesh, 3, eps=0.05, noise=0.01, h=h))
    v = fi.random_direction(mesh.n_total, 4)
    rows = sampled_rows(mesh.n_total, 2000, 5)
    zt, vt = dev(z), dev(v)
    e_ref = ref.energy(z)                      # full-size energy (compensated sum)
    assert abs(prob.energy(zt).item() - e_ref) <= TOL * abs(e_ref)
    for bc in (False, True):
        r = prob.residual(zt, bc=bc).cpu().numpy()
        rr = ref.residual_rows(z, rows, bc=bc)
        assert np.abs(r[rows] - rr).max() <= TOL * np.abs(r).max()
        e1, r1 = prob.energy_residual(zt, bc=bc)     # one-pass value and gradient
        assert abs(e1.item() - e_ref) <= TOL * abs(e_ref)
        assert np.abs(r1.cpu().numpy()[rows] - rr).max() <= TOL * np.abs(r).max()
        y = prob.hvp(zt, vt, bc=bc).cpu().numpy()
        yr = ref.hvp_rows(z, v, rows, bc=bc)
        assert np.abs(y[rows] - yr).max() <= TOL * np.abs(y).max()
        prob.linearize(zt)
        for f in (fem.DETERMINISTIC, fem.BASELINE_SCATTER, fem.LINEARIZED, fem.STREAM_GEOM, fem.REFERENCE_METRIC,
                  fem.COLORED_SCATTER, fem.TILE_COLORED):  # other HVP modes
            yf = prob.hvp(zt, vt, bc=bc, flags=f).cpu().numpy()
            assert np.abs(yf[rows] - yr).max() <= TOL * np.abs(y).max()
        for f in (fem.STREAM_GEOM, fem.REFERENCE_METRIC, fem.COLORED_SCATTER, fem.TILE_COLORED):   # other residual modes
            rf = prob.residual(zt, bc=bc, flags=f).cpu().numpy()
            assert np.abs(rf[rows] - rr).max() <= TOL * np.abs(r).max()
    # tangent and residual patch tests at full size (exact on any P1 mesh)
    dim = mesh.dim
    F = np.diag([1.05] + [0.98] * (dim - 1))
    u_hom = fi.affine_field(mesh, F - np.eye(dim))
    interior = ~fi.boundary_node_mask(mesh)
    r = prob.residual(dev(u_hom)).cpu().numpy().reshape(-1, dim)
    assert np.abs(r[interior]).max() <= 1e-12 * np.abs(r).max()
    w = fi.affine_field(mesh, np.random.default_rng(1).uniform(-1, 1, (dim, dim)))
    y = prob.hvp(dev(u_hom), dev(w)).cpu().numpy().reshape(-1, dim)
    assert np.abs(y[interior]).max() <= 1e-12 * np.abs(y).max()
    # CSR rows, all three modes, vs the oracle's element-Hessian rows
    rp, ci = prob.sparsity()
    rp_n, ci_n = rp.cpu().numpy(), ci.cpu().numpy()
    assert rp_n[-1] == {2: 13973156, 3: 459889659}[cfg]       # SURVEY §8 closed-form nnz
    colors, nc = prob.color()
    assert nc == {2: 18, 3: 90}[cfg]     # cfg 3 count pinned by the oracle in the test below
    srow = sampled_rows(mesh.n_total, 300, 6)
    ref_vals = ref.csr_rows(z, srow, rp_n, ci_n, bc=True)
    idx = np.concatenate([np.arange(rp_n[r], rp_n[r + 1]) for r in srow])
    for mode in ("rows", "batched", "scatter", "colored"):
        vals = prob.assemble_csr(zt, bc=True, mode=mode).cpu().numpy()
        assert np.abs(vals[idx] - ref_vals).max() <= TOL * np.abs(vals).max()
        del vals
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfg", [2, 3])
def test_full_size_coloring_bit_exact(fem, oracle_mod, cfg):
    mesh = fi.config_mesh(cfg)
    prob = fem.Problem(mesh)
    ref = oracle_mod.Oracle(mesh)
    colors, nc = prob.color()
    rcol, rnc = ref.colors()
    assert nc == rnc == {2: 18, 3: 90}[cfg]
    assert np.array_equal(colors.cpu().numpy(), rcol)


def test_full_size_mpc_coloring_bit_exact(fem, oracle_mod):
    mesh = fi.config_mesh(5, n=223)   # ~1e5 DOFs, DOF-level generic path (multipliers)
    prob = fem.Problem(mesh)
    ref = oracle_mod.Oracle(mesh)
    rp, ci = prob.sparsity()
    rrp, rci = ref.sparsity()
    assert np.array_equal(rp.cpu().numpy(), rrp) and np.array_equal(ci.cpu().numpy(), rci)
    colors, nc = prob.color()
    rcol, rnc = ref.colors()
    assert nc == rnc and np.array_equal(colors.cpu().numpy(), rcol)
    z = fi.generic_state(mesh, 3)
    assert rel(prob.assemble_csr(dev(z)), ref.assemble_elem(z)) <= TOL


def test_full_size_newton_cfg2_closed_form(fem, oracle_mod):
    # C15: roller stretch eps = 0.1 has the homogeneous solution u = (F - I) X on any mesh,
    # so the full-size solution must be affine with the oracle's s from a small mesh.
    small = fi.roller_bc(fi.perturb(fi.grid_tri3(8, 8), 0.2, 11).copy_with(material=1), 0.1)
    zs, _ = oracle_mod.Oracle(small).newton(fi.lift(small), cg_rtol=1e-13)
    s_ref = 1.0 + zs.reshape(-1, 2)[:, 1] @ small.coords[:, 1] / (small.coords[:, 1] @ small.coords[:, 1])
    mesh = fi.config_mesh(2)
    prob = fem.Problem(mesh)
    # one load step from the affine predictor u = (eps X, 0) (it satisfies the BCs); the
    # bare lift would stretch the last element column by eps/h = 70x, where the NH tangent
    # is indefinite (c1 = mu - lambda ln J < 0) and CG breaks down.
    z0 = fi.lift(mesh, fi.affine_field(mesh, np.diag([0.1, 0.0])))
    z, info = prob.newton_solve(dev(z0), op=0, cg_rtol=1e-11, rtol=1e-10, atol=1e-14)
    assert info["converged"]
    U = z.cpu().numpy().reshape(-1, 2)
    s = 1.0 + U[:, 1] @ mesh.coords[:, 1] / (mesh.coords[:, 1] @ mesh.coords[:, 1])
    ref = fi.affine_field(mesh, np.diag([0.1, s - 1.0]))
    assert rel(z, ref) <= 1e-10
    assert abs(s - s_ref) < 1e-10


@pytest.mark.parametrize("variant", ["pull", "fused"])
def test_row_assembly_fallback_kernels(fem, oracle_mod, variant, monkeypatch):
    """The row-form fallbacks the node tiles hand over to (meshes the tile plan does not
    cover): the direct-load row pull over HBM context records (FEM_ROWS_PULL) and the
    per-lane-context warp pull (FEM_ROWS_PULL + FEM_ROWS_LEGACY); plans are built per
    problem, so the variables are read when the problem first assembles."""
    monkeypatch.setenv("FEM_ROWS_PULL", "1")
    if variant == "fused":
        monkeypatch.setenv("FEM_ROWS_LEGACY", "1")
    for name in ("3d-nh", "3d-nh-shuffled", "2d-nh-roller", "2d-nh-phases-fext"):
        mesh = MESHES[name]
        z = fi.lift(mesh, fi.generic_state(mesh, 1))
        prob = fem.Problem(mesh)
        for bc in (False, True):
            vals = prob.assemble_csr(dev(z), bc=bc, mode="rows")
            assert rel(vals, oracle_mod.Oracle(mesh).assemble_alg2(z, bc=bc)) <= TOL


def test_row_tiles_32_lanes(fem, oracle_mod, monkeypatch):
    """The 32-lane node tiles (one node per warp, 8-node tiles, each lane summing slots ql and
    ql + 32: the unstructured-mesh form) forced on meshes the 8/16-lane tiles would take,
    incl. multiplier columns; the Delaunay meshes run them by default (> 16 slots, and > 32
    on the graded mesh's surface nodes: two slot passes)."""
    monkeypatch.setenv("FEM_RT_LPN32", "1")
    for name in ("3d-nh", "3d-le", "2d-nh-roller", "2d-le-mpc", "2d-nh-phases-fext"):
        mesh = MESHES[name]
        z = fi.lift(mesh, fi.generic_state(mesh, 1))
        prob = fem.Problem(mesh)
        for bc in (False, True):
            vals = prob.assemble_csr(dev(z), bc=bc, mode="rows")
            assert rel(vals, oracle_mod.Oracle(mesh).assemble_alg2(z, bc=bc)) <= TOL


def test_row_tiles_soa_records(fem, oracle_mod, monkeypatch):
    """The conflict-free SoA record layout of the 3D node tiles (FEM_RT_SOA=1 at run time:
    4-colored tile elements, color-distinct co-schedules from first fit or the plan's
    depth-first search, idle steps without loads) against the oracle's Alg. 2 CSR, with and
    without BC, on the structured, shuffled and LE 3D meshes; 2D meshes keep the odd-stride
    records."""
    monkeypatch.setenv("FEM_RT_SOA", "1")
    for name in ("3d-nh", "3d-le", "3d-nh-shuffled", "2d-nh-roller"):
        mesh = MESHES[name]
        z = fi.lift(mesh, fi.generic_state(mesh, 1))
        prob = fem.Problem(mesh)
        for bc in (False, True):
            vals = prob.assemble_csr(dev(z), bc=bc, mode="rows")
            assert rel(vals, oracle_mod.Oracle(mesh).assemble_alg2(z, bc=bc)) <= TOL
    mesh = fi.config_mesh(3, n=24)  # several hundred tiles: the plan's DFS co-schedules run
    z = fi.lift(mesh, fi.generic_state(mesh, 2))
    monkeypatch.setenv("FEM_RT_SOA", "0")
    ref = fem.Problem(mesh).assemble_csr(dev(z), bc=True, mode="rows")
    monkeypatch.setenv("FEM_RT_SOA", "1")
    vals = fem.Problem(mesh).assemble_csr(dev(z), bc=True, mode="rows")
    assert rel(vals, ref.cpu().numpy()) <= TOL


def test_cg_graph_batches_match_direct_launches(fem, monkeypatch):
    """CG iterations between host checks run as a captured CUDA graph (check_every >= 2);
    with the deterministic CSR operator the iterates equal the directly launched ones bit
    for bit (the HVP's tile-boundary REDs make it run-to-run reproducible only to rounding)."""
    mesh = MESHES["3d-nh"]
    z = dev(fi.lift(mesh, fi.generic_state(mesh, 1)))
    b = fi.random_direction(mesh.n_total, 2)
    b[mesh.dirichlet_dofs] = 0.0
    prob = fem.Problem(mesh)
    vals = prob.assemble_csr(z, bc=True)
    xg, ig = prob.cg_solve(dev(b), vals=vals, op=1, rtol=1e-12, check_every=8)
    hg, hig = prob.cg_solve(dev(b), z=z, op=0, rtol=1e-12, check_every=8)
    monkeypatch.setenv("FEM_NO_GRAPHS", "1")
    xd, idd = prob.cg_solve(dev(b), vals=vals, op=1, rtol=1e-12, check_every=8)
    hd, hid = prob.cg_solve(dev(b), z=z, op=0, rtol=1e-12, check_every=8)
    assert ig["converged"] and idd["converged"] and ig["iters"] == idd["iters"]
    assert torch.equal(xg, xd)
    assert hig["converged"] and hid["converged"]
    assert rel(hg, hd.cpu().numpy()) <= 1e-10


def test_linearized_hvp_and_newton(fem, monkeypatch):
    """fem_linearize caches the metric-form tangent at z; FEM_LINEARIZED HVPs equal the full
    HVP, and Newton-Krylov linearizing at every iterate (default) reaches the same solution
    as recomputing the state per HVP (FEM_NEWTON_RECOMPUTE)."""
    for name in ("3d-nh", "2d-nh-roller", "2d-nh-phases-fext"):
        mesh = MESHES[name]
        z = dev(fi.lift(mesh, fi.generic_state(mesh, 1)))
        v = dev(fi.random_direction(mesh.n_total, 2))
        prob = fem.Problem(mesh)
        prob.linearize(z)
        for bc in (False, True):
            y = prob.hvp(z, v, bc=bc)
            yl = prob.hvp(z, v, bc=bc, flags=fem.LINEARIZED)
            assert rel(yl, y.cpu().numpy()) <= 1e-13
    mesh = MESHES["3d-nh"]
    prob = fem.Problem(mesh)
    z0 = dev(fi.lift(mesh))
    za, ia = prob.newton_solve(z0, cg_rtol=1e-12, check_every=8)
    monkeypatch.setenv("FEM_NEWTON_RECOMPUTE", "1")
    zb, ib = prob.newton_solve(z0, cg_rtol=1e-12, check_every=8)
    assert ia["converged"] and ib["converged"]
    assert rel(za, zb.cpu().numpy()) <= 1e-10
