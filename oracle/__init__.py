"""ctypes binding of the CPU oracle (liboracle.so).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path (paper_2602_12365_b200) never does.
All arrays are host numpy arrays; see oracle/oracle.h for argument meanings and
oracle/oracle.c for the paper passages each function follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

STATUS = {0: "OK", 1: "INVALID_ARG", 2: "DEGENERATE_ELEMENT", 3: "INVERTED_ELEMENT",
          4: "NONFINITE", 5: "CG_BREAKDOWN", 6: "NOT_CONVERGED", 8: "OUT_OF_MEMORY"}
APPLY_BC = 1


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {STATUS.get(status, status)}")
        self.status = status


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, -O2 -ffp-contract=off, single thread)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-Wall", "-o", _SO, src, "-lm"])
    return _SO


class _Mesh(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_nodes", C.c_int64), ("n_elems", C.c_int64),
                ("coords", C.c_void_p), ("conn", C.c_void_p), ("material", C.c_int),
                ("lam", C.c_double), ("mu", C.c_double), ("phase", C.c_void_p),
                ("lambda_tab", C.c_void_p), ("mu_tab", C.c_void_p), ("n_phases", C.c_int),
                ("n_dirichlet", C.c_int64), ("dirichlet_dofs", C.c_void_p),
                ("dirichlet_vals", C.c_void_p), ("n_mpc", C.c_int64), ("mpc_slave", C.c_void_p),
                ("mpc_master", C.c_void_p), ("mpc_offset", C.c_void_p), ("f_ext", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_SO)
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


class Oracle:
    """Holds contiguous copies of a fem_inputs.Mesh and calls fem_ref_* on them."""

    def __init__(self, mesh):
        self.mesh = mesh
        keep = {}

        def arr(x, dt):
            if x is None:
                return None
            a = np.ascontiguousarray(x, dtype=dt)
            keep[id(a)] = a
            return a

        self._coords = arr(mesh.coords, np.float64)
        self._conn = arr(mesh.conn, np.int32)
        self._dd = arr(mesh.dirichlet_dofs, np.int32)
        self._dv = arr(mesh.dirichlet_vals, np.float64)
        self._ms = arr(mesh.mpc_slave, np.int32)
        self._mm = arr(mesh.mpc_master, np.int32)
        self._mo = arr(mesh.mpc_offset, np.float64)
        self._fe = arr(mesh.f_ext, np.float64)
        self._ph = arr(mesh.phase, np.uint8)
        self._lt = arr(mesh.lambda_tab, np.float64)
        self._mt = arr(mesh.mu_tab, np.float64)
        self._keep = keep
        self.s = _Mesh(mesh.dim, mesh.n_nodes, mesh.n_elems, _p(self._coords), _p(self._conn),
                       mesh.material, mesh.lam, mesh.mu, _p(self._ph), _p(self._lt), _p(self._mt),
                       0 if self._lt is None else len(self._lt), len(self._dd), _p(self._dd),
                       _p(self._dv), len(self._ms), _p(self._ms), _p(self._mm), _p(self._mo),
                       _p(self._fe))
        self.N = mesh.n_total
        self._pattern = None
        self._colors = None

    def _call(self, name, *args):
        st = getattr(lib(), name)(C.byref(self.s), *args)
        if st != 0:
            raise OracleError(st, name)

    @staticmethod
    def _f64(x):
        return np.ascontiguousarray(x, dtype=np.float64)

    # -- energy and derivatives -------------------------------------------------------
    def geometry(self):
        d, E = self.mesh.dim, self.mesh.n_elems
        G = np.empty((E, d + 1, d))
        vol = np.empty(E)
        self._call("fem_ref_geometry", C.c_void_p(G.ctypes.data), C.c_void_p(vol.ctypes.data))
        return G, vol

    def energy(self, z) -> float:
        z = self._f64(z)
        out = C.c_double(0.0)
        self._call("fem_ref_energy", C.c_void_p(z.ctypes.data), C.byref(out))
        return out.value

    def residual(self, z, bc: bool = False):
        z = self._f64(z)
        r = np.empty(self.N)
        self._call("fem_ref_residual", C.c_void_p(z.ctypes.data), C.c_void_p(r.ctypes.data),
                   C.c_uint(APPLY_BC if bc else 0))
        return r

    def hvp(self, z, v, bc: bool = False):
        z, v = self._f64(z), self._f64(v)
        y = np.empty(self.N)
        self._call("fem_ref_hvp", C.c_void_p(z.ctypes.data), C.c_void_p(v.ctypes.data),
                   C.c_void_p(y.ctypes.data), C.c_uint(APPLY_BC if bc else 0))
        return y

    def dense_hessian(self, z, bc: bool = False):
        z = self._f64(z)
        H = np.empty((self.N, self.N))
        self._call("fem_ref_dense_hessian", C.c_void_p(z.ctypes.data), C.c_void_p(H.ctypes.data),
                   C.c_uint(APPLY_BC if bc else 0))
        return H

    def residual_rows(self, z, rows, bc: bool = False):
        z = self._f64(z)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty(len(rows))
        self._call("fem_ref_residual_rows", C.c_void_p(z.ctypes.data), C.c_int64(len(rows)),
                   C.c_void_p(rows.ctypes.data), C.c_void_p(out.ctypes.data),
                   C.c_uint(APPLY_BC if bc else 0))
        return out

    def hvp_rows(self, z, v, rows, bc: bool = False):
        z, v = self._f64(z), self._f64(v)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty(len(rows))
        self._call("fem_ref_hvp_rows", C.c_void_p(z.ctypes.data), C.c_void_p(v.ctypes.data),
                   C.c_int64(len(rows)), C.c_void_p(rows.ctypes.data),
                   C.c_void_p(out.ctypes.data), C.c_uint(APPLY_BC if bc else 0))
        return out

    # -- pattern, coloring, assembly --------------------------------------------------
    def sparsity(self):
        if self._pattern is None:
            row_ptr = np.empty(self.N + 1, np.int64)
            self._call("fem_ref_sparsity", C.c_void_p(row_ptr.ctypes.data), C.c_void_p(None))
            col = np.empty(int(row_ptr[-1]), np.int32)
            self._call("fem_ref_sparsity", C.c_void_p(row_ptr.ctypes.data),
                       C.c_void_p(col.ctypes.data))
            self._pattern = (row_ptr, col)
        return self._pattern

    def colors(self):
        if self._colors is None:
            rp, ci = self.sparsity()
            self._colors = color(rp, ci)
        return self._colors

    def assemble_alg2(self, z, bc: bool = False):
        rp, ci = self.sparsity()
        colors, nc = self.colors()
        z = self._f64(z)
        vals = np.empty(len(ci))
        self._call("fem_ref_assemble_alg2", C.c_void_p(z.ctypes.data), C.c_void_p(rp.ctypes.data),
                   C.c_void_p(ci.ctypes.data), C.c_void_p(colors.ctypes.data), C.c_int32(nc),
                   C.c_void_p(vals.ctypes.data), C.c_uint(APPLY_BC if bc else 0))
        return vals

    def assemble_elem(self, z, bc: bool = False):
        rp, ci = self.sparsity()
        z = self._f64(z)
        vals = np.empty(len(ci))
        self._call("fem_ref_assemble_elem", C.c_void_p(z.ctypes.data), C.c_void_p(rp.ctypes.data),
                   C.c_void_p(ci.ctypes.data), C.c_void_p(vals.ctypes.data),
                   C.c_uint(APPLY_BC if bc else 0))
        return vals

    def csr_rows(self, z, rows, row_ptr, col_idx, bc: bool = False):
        z = self._f64(z)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        n_out = int(np.sum(rp[rows + 1] - rp[rows]))
        out = np.empty(n_out)
        self._call("fem_ref_csr_rows", C.c_void_p(z.ctypes.data), C.c_void_p(rp.ctypes.data),
                   C.c_void_p(ci.ctypes.data), C.c_int64(len(rows)), C.c_void_p(rows.ctypes.data),
                   C.c_void_p(out.ctypes.data), C.c_uint(APPLY_BC if bc else 0))
        return out

    # -- solvers ----------------------------------------------------------------------
    def cg(self, b, x0=None, op: int = 0, z=None, vals=None, rtol=1e-10, atol=0.0,
           max_iter=10000, row_ptr=None, col_idx=None):
        b = self._f64(b)
        x = np.zeros(self.N) if x0 is None else np.array(x0, np.float64, copy=True)
        zz = self._f64(np.zeros(self.N) if z is None else z)
        rp = ci = None
        if op == 1:
            rp, ci = self.sparsity() if row_ptr is None else (
                np.ascontiguousarray(row_ptr, np.int64), np.ascontiguousarray(col_idx, np.int32))
            vals = self._f64(vals)
        iters, r0, r1 = C.c_int(0), C.c_double(0), C.c_double(0)
        st = lib().fem_ref_cg(C.byref(self.s), C.c_int(op), C.c_void_p(zz.ctypes.data),
                              C.c_void_p(_p(rp)), C.c_void_p(_p(ci)), C.c_void_p(_p(vals)),
                              C.c_void_p(b.ctypes.data), C.c_void_p(x.ctypes.data),
                              C.c_double(rtol), C.c_double(atol), C.c_int(max_iter),
                              C.byref(iters), C.byref(r0), C.byref(r1))
        return x, {"status": st, "iters": iters.value, "res0": r0.value, "res": r1.value}

    def newton(self, z0, atol=1e-12, rtol=1e-10, max_iter=50, cg_rtol=1e-10, cg_max_iter=100000):
        z = np.array(z0, np.float64, copy=True)
        it, cgt, r0, r1 = C.c_int(0), C.c_int(0), C.c_double(0), C.c_double(0)
        st = lib().fem_ref_newton(C.byref(self.s), C.c_void_p(z.ctypes.data), C.c_double(atol),
                                  C.c_double(rtol), C.c_int(max_iter), C.c_double(cg_rtol),
                                  C.c_int(cg_max_iter), C.byref(it), C.byref(cgt), C.byref(r0),
                                  C.byref(r1))
        return z, {"status": st, "iters": it.value, "cg_iters": cgt.value, "res0": r0.value,
                   "res": r1.value}


    def mean_stress(self, z):
        """(volume average of P as a dim x dim array, |Omega|) — fem_ref_mean_stress."""
        z = self._f64(z)
        d = self.mesh.dim
        sig = np.zeros(d * d)
        vol = C.c_double(0)
        st = lib().fem_ref_mean_stress(C.byref(self.s), C.c_void_p(z.ctypes.data),
                                       C.c_void_p(sig.ctypes.data), C.byref(vol))
        if st:
            raise OracleError(st, "fem_ref_mean_stress")
        return sig.reshape(d, d), vol.value

    def traction_load(self, facets, traction):
        """int N_a t dGamma over the facets (fem_ref_traction_load), [N_u]."""
        f = np.zeros(self.mesh.n_nodes * self.mesh.dim)
        fa = np.ascontiguousarray(facets, np.int32)
        t = np.asarray(traction, np.float64)
        t = np.ascontiguousarray(np.tile(t, (len(fa), 1)) if t.ndim == 1 else t)
        st = lib().fem_ref_traction_load(C.c_int(self.mesh.dim), C.c_int64(self.mesh.n_nodes),
                                         C.c_void_p(self._coords.ctypes.data), C.c_int64(len(fa)),
                                         C.c_void_p(fa.ctypes.data), C.c_void_p(t.ctypes.data),
                                         C.c_void_p(f.ctypes.data))
        if st:
            raise OracleError(st, "fem_ref_traction_load")
        return f

    def body_load(self, b):
        f = np.zeros(self.mesh.n_nodes * self.mesh.dim)
        bb = np.ascontiguousarray(np.asarray(b, np.float64))
        st = lib().fem_ref_body_load(C.byref(self.s), C.c_void_p(bb.ctypes.data),
                                     C.c_void_p(f.ctypes.data))
        if st:
            raise OracleError(st, "fem_ref_body_load")
        return f

    def newton_dense(self, z0, atol=1e-12, rtol=1e-10, max_iter=50):
        """Full-step Newton on the BC-applied Lagrangian with the dense Hessian and
        numpy.linalg.solve for each step — the plain definition of the stationary point of
        L (saddle points included) for small N (O-dense, N <= ~2000)."""
        z = np.array(z0, np.float64, copy=True)
        r0 = None
        for it in range(max_iter + 1):
            r = self.residual(z, bc=True)
            nr = float(np.linalg.norm(r))
            r0 = nr if r0 is None else r0
            if nr <= max(atol, rtol * r0):
                return z, {"iters": it, "res0": r0, "res": nr, "converged": True}
            if it == max_iter:
                break
            z += np.linalg.solve(self.dense_hessian(z, bc=True), -r)
        return z, {"iters": max_iter, "res0": r0, "res": nr, "converged": False}


class _Vw(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_nodes", C.c_int64), ("n_elems", C.c_int64),
                ("coords", C.c_void_p), ("conn", C.c_void_p), ("diffusivity", C.c_double),
                ("velocity", C.c_void_p), ("mass_coef", C.c_double), ("n_dirichlet", C.c_int64),
                ("dirichlet_nodes", C.c_void_p), ("dirichlet_vals", C.c_void_p)]


class VwOracle:
    """Virtual-work path (f4): fem_ref_vw_residual / fem_ref_vw_jvp on host arrays."""

    def __init__(self, coords, conn, diffusivity, velocity, mass_coef=0.0, dirichlet_nodes=None,
                 dirichlet_vals=None):
        self.coords = np.ascontiguousarray(coords, np.float64)
        self.conn = np.ascontiguousarray(conn, np.int32)
        self.vel = np.ascontiguousarray(velocity, np.float64)
        dn = np.zeros(0, np.int32) if dirichlet_nodes is None else dirichlet_nodes
        dv = np.zeros(0) if dirichlet_vals is None else dirichlet_vals
        self.dn = np.ascontiguousarray(dn, np.int32)
        self.dv = np.ascontiguousarray(dv, np.float64)
        self.n = self.coords.shape[0]
        self.s = _Vw(self.coords.shape[1], self.n, self.conn.shape[0], _p(self.coords),
                     _p(self.conn), diffusivity, _p(self.vel), mass_coef, len(self.dn),
                     _p(self.dn), _p(self.dv))

    def residual(self, c, c_old=None, bc=False):
        c = np.ascontiguousarray(c, np.float64)
        co = None if c_old is None else np.ascontiguousarray(c_old, np.float64)
        r = np.zeros(self.n)
        st = lib().fem_ref_vw_residual(C.byref(self.s), C.c_void_p(c.ctypes.data),
                                       C.c_void_p(_p(co)), C.c_void_p(r.ctypes.data),
                                       C.c_uint(APPLY_BC if bc else 0))
        if st:
            raise OracleError(st, "fem_ref_vw_residual")
        return r

    def jvp(self, x, bc=False):
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n)
        st = lib().fem_ref_vw_jvp(C.byref(self.s), C.c_void_p(x.ctypes.data),
                                  C.c_void_p(y.ctypes.data), C.c_uint(APPLY_BC if bc else 0))
        if st:
            raise OracleError(st, "fem_ref_vw_jvp")
        return y

    def dense(self, bc=False):
        """K column by column (n JVPs) — the plain definition for small n."""
        return np.stack([self.jvp(np.eye(self.n)[j], bc=bc) for j in range(self.n)], axis=1)


def color(row_ptr, col_idx):
    """Distance-2 greedy coloring of an arbitrary CSR pattern (fem_ref_color)."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    n = len(rp) - 1
    colors = np.empty(n, np.int32)
    nc = C.c_int32(0)
    st = lib().fem_ref_color(C.c_int64(n), C.c_void_p(rp.ctypes.data), C.c_void_p(ci.ctypes.data),
                             C.c_void_p(colors.ctypes.data), C.byref(nc))
    if st != 0:
        raise OracleError(st, "fem_ref_color")
    return colors, nc.value


def spmv(row_ptr, col_idx, vals, x):
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int32)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(len(rp) - 1)
    lib().fem_ref_spmv(C.c_int64(len(rp) - 1), C.c_void_p(rp.ctypes.data),
                       C.c_void_p(ci.ctypes.data), C.c_void_p(v.ctypes.data),
                       C.c_void_p(xx.ctypes.data), C.c_void_p(y.ctypes.data))
    return y


class _Dummy:
    """Mesh stand-in with N = n unknowns and no elements, for CG on a given CSR."""

    def __init__(self, n):
        self.dim, self.coords = 1, np.zeros((n, 1))
        self.conn = np.zeros((0, 2), np.int32)
        self.material, self.lam, self.mu = 0, 0.0, 0.0
        self.dirichlet_dofs = np.zeros(0, np.int32)
        self.dirichlet_vals = np.zeros(0)
        self.mpc_slave = self.mpc_master = np.zeros(0, np.int32)
        self.mpc_offset = np.zeros(0)
        self.f_ext = self.phase = self.lambda_tab = self.mu_tab = None
        self.n_nodes, self.n_elems, self.n_total = n, 0, n


def cg_csr(row_ptr, col_idx, vals, b, x0=None, rtol=1e-10, atol=0.0, max_iter=10000):
    """fem_ref_cg with op 1 on an arbitrary CSR matrix."""
    o = Oracle(_Dummy(len(row_ptr) - 1))
    return o.cg(b, x0=x0, op=1, vals=vals, rtol=rtol, atol=atol, max_iter=max_iter,
                row_ptr=row_ptr, col_idx=col_idx)
