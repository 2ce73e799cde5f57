"""Thin ctypes binding of libfem.so (include/fem.h) — argument marshalling only.

Every computation runs in the library's sm_100a kernels; PyTorch provides device memory
and the current CUDA stream.  There is no CPU fallback: if libfem.so is missing or no
CUDA device is present the calls raise.

The names follow the C ABI: Problem.energy -> fem_energy, .residual -> fem_residual,
.hvp -> fem_hvp, .sparsity -> fem_sparsity, .color -> fem_color,
.assemble_csr -> fem_assemble_csr, .spmv -> fem_spmv, .cg_solve -> fem_cg_solve,
.minres_solve -> fem_minres_solve, .mean_stress -> fem_mean_stress,
.newton_solve -> fem_newton_solve.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfem.so")

APPLY_BC = 1
DETERMINISTIC = 2
ASSEMBLE_LITERAL = 4
ASSEMBLE_JCOMP = 32
ASSEMBLE_ROWS = 64
ASSEMBLE_SCATTER = 128
ASSEMBLE_COLORED = 4096
LINEARIZED = 256
BASELINE_SCATTER = 8
STREAM_GEOM = 512          # residual / HVP from the streamed per-element geometry (Alg. 1)
COLORED_SCATTER = 1024     # residual / HVP by element-colored conflict-free passes
TILE_COLORED = 2048        # residual / HVP by tile-colored passes (plain boundary writes)
REFERENCE_METRIC = 8192    # NH residual / HVP: read the cached reference metric (Alg. 1)
LOCAL_ONLY = 16
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "DEGENERATE_ELEMENT", 3: "INVERTED_ELEMENT",
          4: "NONFINITE", 5: "CG_BREAKDOWN", 6: "NOT_CONVERGED", 7: "TOO_MANY_COLORS",
          8: "OUT_OF_MEMORY", 9: "CUDA", 10: "NCCL"}

# every symbol include/fem.h declares (checked by tests/test_abi.py)
EXPORTS = ("fem_create", "fem_destroy", "fem_query", "fem_check", "fem_apply_dirichlet",
           "fem_energy", "fem_residual", "fem_energy_residual", "fem_hvp", "fem_sparsity", "fem_color",
           "fem_assemble_csr", "fem_spmv", "fem_cg_solve", "fem_minres_solve",
           "fem_mean_stress", "fem_linearize", "fem_add_traction", "fem_add_body_force", "fem_get_fext",
           "fem_newton_solve", "fem_vw_create", "fem_vw_destroy", "fem_vw_apply_dirichlet",
           "fem_vw_residual", "fem_vw_jvp", "fem_vw_gmres_solve",
           "fem_nccl_unique_id", "fem_nccl_comm_init", "fem_nccl_comm_destroy", "fem_nccl_comm_count",
           "fem_allreduce_sum", "fem_halo_size", "fem_halo_pack", "fem_halo_combine",
           "fem_last_error", "fem_version")


class FemError(RuntimeError):
    def __init__(self, status: int, what: str, msg: str = ""):
        super().__init__(f"{what}: {STATUS.get(status, status)} {msg}".strip())
        self.status = status


class MeshDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_nodes", C.c_int64), ("n_elems", C.c_int64),
                ("coords", C.c_void_p), ("conn", C.c_void_p), ("material", C.c_int),
                ("lam", C.c_double), ("mu", C.c_double), ("phase", C.c_void_p),
                ("lambda_tab", C.c_void_p), ("mu_tab", C.c_void_p), ("n_phases", C.c_int),
                ("n_dirichlet", C.c_int64), ("dirichlet_dofs", C.c_void_p),
                ("dirichlet_vals", C.c_void_p), ("n_mpc", C.c_int64), ("mpc_slave", C.c_void_p),
                ("mpc_master", C.c_void_p), ("mpc_offset", C.c_void_p), ("f_ext", C.c_void_p)]


class DistDesc(C.Structure):
    _fields_ = [("nccl_comm", C.c_void_p), ("rank", C.c_int), ("size", C.c_int),
                ("n_nbr", C.c_int), ("nbr_rank", C.c_void_p), ("nbr_offset", C.c_void_p),
                ("nbr_nodes", C.c_void_p), ("owned", C.c_void_p)]


class CgOpts(C.Structure):
    _fields_ = [("op", C.c_int), ("rtol", C.c_double), ("atol", C.c_double),
                ("max_iter", C.c_int), ("jacobi", C.c_int), ("check_every", C.c_int),
                ("hvp_flags", C.c_uint)]


class CgReport(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("res0", C.c_double),
                ("res", C.c_double)]


class VwDesc(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_nodes", C.c_int64), ("n_elems", C.c_int64),
                ("coords", C.c_void_p), ("conn", C.c_void_p), ("diffusivity", C.c_double),
                ("velocity", C.c_void_p), ("mass_coef", C.c_double), ("n_dirichlet", C.c_int64),
                ("dirichlet_nodes", C.c_void_p), ("dirichlet_vals", C.c_void_p)]


class GmresOpts(C.Structure):
    _fields_ = [("restart", C.c_int), ("max_iter", C.c_int), ("rtol", C.c_double),
                ("atol", C.c_double)]


class NewtonOpts(C.Structure):
    _fields_ = [("atol", C.c_double), ("rtol", C.c_double), ("max_iter", C.c_int),
                ("cg", CgOpts), ("forcing", C.c_double)]


class NewtonReport(C.Structure):
    _fields_ = [("iters", C.c_int), ("cg_iters", C.c_int), ("converged", C.c_int),
                ("res0", C.c_double), ("res", C.c_double)]


_lib = None


def load_library():
    """Load libfem.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(LIB_PATH)
        for name in EXPORTS:
            getattr(lib, name)  # AttributeError if an export is missing
        vp, i64p = C.c_void_p, C.POINTER(C.c_int64)
        lib.fem_create.argtypes = [C.POINTER(vp), C.POINTER(MeshDesc), C.POINTER(DistDesc), vp]
        lib.fem_destroy.argtypes = [vp]
        lib.fem_query.argtypes = [vp, i64p, i64p, C.POINTER(C.c_int32)]
        lib.fem_check.argtypes = [vp, vp]
        lib.fem_apply_dirichlet.argtypes = [vp, vp, vp]
        lib.fem_energy.argtypes = [vp, vp, vp, vp]
        lib.fem_residual.argtypes = [vp, vp, vp, C.c_uint, vp]
        lib.fem_energy_residual.argtypes = [vp, vp, vp, vp, C.c_uint, vp]
        lib.fem_hvp.argtypes = [vp, vp, vp, vp, C.c_uint, vp]
        lib.fem_sparsity.argtypes = [vp, vp, vp, vp]
        lib.fem_color.argtypes = [vp, vp, C.POINTER(C.c_int32), vp]
        lib.fem_assemble_csr.argtypes = [vp, vp, vp, C.c_uint, vp]
        lib.fem_spmv.argtypes = [vp, vp, vp, vp, vp]
        lib.fem_cg_solve.argtypes = [vp, vp, vp, vp, vp, C.POINTER(CgOpts), C.POINTER(CgReport), vp]
        lib.fem_minres_solve.argtypes = [vp, vp, vp, vp, vp, C.POINTER(CgOpts), C.POINTER(CgReport), vp]
        lib.fem_linearize.argtypes = [vp, vp, vp]
        lib.fem_mean_stress.argtypes = [vp, vp, C.POINTER(C.c_double), C.POINTER(C.c_double), vp]
        lib.fem_add_traction.argtypes = [vp, C.c_int64, vp, vp, vp]
        lib.fem_add_body_force.argtypes = [vp, C.POINTER(C.c_double), vp]
        lib.fem_get_fext.argtypes = [vp, vp, vp]
        lib.fem_vw_create.argtypes = [C.POINTER(vp), C.POINTER(VwDesc), vp]
        lib.fem_vw_destroy.argtypes = [vp]
        lib.fem_vw_apply_dirichlet.argtypes = [vp, vp, vp]
        lib.fem_vw_residual.argtypes = [vp, vp, vp, vp, C.c_uint, vp]
        lib.fem_vw_jvp.argtypes = [vp, vp, vp, C.c_uint, vp]
        lib.fem_vw_gmres_solve.argtypes = [vp, vp, vp, C.POINTER(GmresOpts), C.POINTER(CgReport), vp]
        lib.fem_newton_solve.argtypes = [vp, vp, C.POINTER(NewtonOpts), C.POINTER(NewtonReport), vp]
        lib.fem_nccl_unique_id.argtypes = [C.c_char_p]
        lib.fem_nccl_comm_init.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(vp)]
        lib.fem_nccl_comm_destroy.argtypes = [vp]
        lib.fem_nccl_comm_count.argtypes = [vp, C.POINTER(C.c_int)]
        lib.fem_allreduce_sum.argtypes = [vp, vp, C.c_int, vp]
        lib.fem_halo_size.argtypes = [vp, i64p]
        lib.fem_halo_pack.argtypes = [vp, vp, vp, vp]
        lib.fem_halo_combine.argtypes = [vp, vp, vp, vp]
        lib.fem_last_error.restype = C.c_char_p
        lib.fem_version.restype = C.c_char_p
        _lib = lib
    return _lib


def _check(st: int, what: str):
    if st != 0:
        raise FemError(st, what, load_library().fem_last_error().decode(errors="replace"))


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    assert t.is_contiguous(), "tensors passed to libfem must be contiguous"
    return t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _dev(x, dtype, device):
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device=device)


class Problem:
    """fem_problem handle for a mesh (fem_inputs.Mesh or any object with its fields)."""

    def __init__(self, mesh, device: str | torch.device = "cuda", plan=None, nccl_comm=None):
        """plan: paper_2602_12365_b200.dist.HaloPlan for a multi-GPU rank (None = one GPU);
        nccl_comm: handle from nccl_comm_init (None: only FEM_LOCAL_ONLY + halo pack/combine)."""
        lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("libfem needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device)
        self.dim = mesh.dim
        f64, i32 = torch.float64, torch.int32
        keep = dict(coords=_dev(mesh.coords, f64, self.device), conn=_dev(mesh.conn, i32, self.device),
                    dd=_dev(mesh.dirichlet_dofs, i32, self.device),
                    dv=_dev(mesh.dirichlet_vals, f64, self.device),
                    ms=_dev(mesh.mpc_slave, i32, self.device), mm=_dev(mesh.mpc_master, i32, self.device),
                    mo=_dev(mesh.mpc_offset, f64, self.device),
                    fe=_dev(getattr(mesh, "f_ext", None), f64, self.device),
                    ph=_dev(getattr(mesh, "phase", None), torch.uint8, self.device))
        lt = getattr(mesh, "lambda_tab", None)
        mt = getattr(mesh, "mu_tab", None)
        self._lt = None if lt is None else np.ascontiguousarray(lt, np.float64)
        self._mt = None if mt is None else np.ascontiguousarray(mt, np.float64)
        n_nodes = int(keep["coords"].shape[0])
        n_elems = int(keep["conn"].shape[0])
        desc = MeshDesc(mesh.dim, n_nodes, n_elems, _ptr(keep["coords"]), _ptr(keep["conn"]),
                        int(mesh.material), float(mesh.lam), float(mesh.mu), _ptr(keep["ph"]),
                        None if self._lt is None else self._lt.ctypes.data,
                        None if self._mt is None else self._mt.ctypes.data,
                        0 if self._lt is None else len(self._lt), int(keep["dd"].numel()),
                        _ptr(keep["dd"]), _ptr(keep["dv"]), int(keep["ms"].numel()),
                        _ptr(keep["ms"]), _ptr(keep["mm"]), _ptr(keep["mo"]), _ptr(keep["fe"]))
        dist = None
        if plan is not None and plan.size > 1:
            self._plan_arrays = (np.ascontiguousarray(plan.nbr_rank, np.int32),
                                 np.ascontiguousarray(plan.nbr_offset, np.int64),
                                 np.ascontiguousarray(plan.nbr_nodes, np.int32),
                                 np.ascontiguousarray(plan.owned, np.uint8))
            nr, no, nn, ow = self._plan_arrays
            dist = DistDesc(nccl_comm, plan.rank, plan.size, len(nr), nr.ctypes.data,
                            no.ctypes.data, nn.ctypes.data if len(nn) else None, ow.ctypes.data)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib.fem_create(C.byref(h), C.byref(desc), C.byref(dist) if dist else None,
                                  _stream()), "fem_create")
        self._h = h
        self.plan = plan
        n = C.c_int64()
        lib.fem_query(h, C.byref(n), None, None)
        self.N = int(n.value)
        self.n_u = n_nodes * mesh.dim

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            try:
                torch.cuda.synchronize(self.device)
            except Exception:
                pass
            _lib.fem_destroy(h)
            self._h = None

    # ---------------------------------------------------------------- helpers
    def _vec(self, x, name="x") -> torch.Tensor:
        t = _dev(x, torch.float64, self.device)
        if t.numel() != self.N:
            raise ValueError(f"{name}: expected {self.N} entries, got {t.numel()}")
        return t

    def _out(self, out, n=None):
        n = self.N if n is None else n
        if out is None:
            return torch.empty(n, dtype=torch.float64, device=self.device)
        assert out.dtype == torch.float64 and out.numel() == n and out.is_contiguous()
        return out

    def query(self):
        n, nnz, nc = C.c_int64(), C.c_int64(), C.c_int32()
        _check(load_library().fem_query(self._h, C.byref(n), C.byref(nnz), C.byref(nc)), "fem_query")
        return n.value, nnz.value, nc.value

    def check(self):
        _check(load_library().fem_check(self._h, _stream()), "fem_check")

    # ---------------------------------------------------------------- hot path
    def apply_dirichlet(self, z: torch.Tensor) -> torch.Tensor:
        _check(load_library().fem_apply_dirichlet(self._h, _ptr(z), _stream()), "fem_apply_dirichlet")
        return z

    def energy(self, z, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        z = self._vec(z, "z")
        out = self._out(out, 1)
        _check(load_library().fem_energy(self._h, _ptr(z), _ptr(out), _stream()), "fem_energy")
        return out

    def residual(self, z, bc: bool = False, out=None, flags: int = 0) -> torch.Tensor:
        z = self._vec(z, "z")
        out = self._out(out)
        _check(load_library().fem_residual(self._h, _ptr(z), _ptr(out), (APPLY_BC if bc else 0) | flags,
                                           _stream()), "fem_residual")
        return out

    def energy_residual(self, z, bc: bool = False, flags: int = 0, out_energy=None, out=None):
        """(energy [1], residual [N]) from one element pass (fem_energy_residual)."""
        z = self._vec(z, "z")
        e = self._out(out_energy, 1)
        r = self._out(out)
        _check(load_library().fem_energy_residual(self._h, _ptr(z), _ptr(e), _ptr(r),
                                                  (APPLY_BC if bc else 0) | flags, _stream()),
               "fem_energy_residual")
        return e, r

    def hvp(self, z, v, bc: bool = False, out=None, flags: int = 0) -> torch.Tensor:
        z, v = self._vec(z, "z"), self._vec(v, "v")
        out = self._out(out)
        _check(load_library().fem_hvp(self._h, _ptr(z), _ptr(v), _ptr(out),
                                      (APPLY_BC if bc else 0) | flags, _stream()), "fem_hvp")
        return out

    def sparsity(self):
        lib = load_library()
        _check(lib.fem_sparsity(self._h, None, None, _stream()), "fem_sparsity")
        _, nnz, _ = self.query()
        rp = torch.empty(self.N + 1, dtype=torch.int64, device=self.device)
        ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=self.device)[:nnz]
        _check(lib.fem_sparsity(self._h, _ptr(rp), _ptr(ci) if nnz else None, _stream()), "fem_sparsity")
        return rp, ci

    def nnz(self) -> int:
        _check(load_library().fem_sparsity(self._h, None, None, _stream()), "fem_sparsity")
        return self.query()[1]

    def color(self):
        colors = torch.empty(self.N, dtype=torch.int32, device=self.device)
        nc = C.c_int32()
        _check(load_library().fem_color(self._h, _ptr(colors), C.byref(nc), _stream()), "fem_color")
        return colors, nc.value

    def assemble_csr(self, z, bc: bool = False, mode: str = "auto", out=None) -> torch.Tensor:
        z = self._vec(z, "z")
        flags = (APPLY_BC if bc else 0) | {"batched": ASSEMBLE_JCOMP, "literal": ASSEMBLE_LITERAL,
                                             "rows": ASSEMBLE_ROWS, "scatter": ASSEMBLE_SCATTER,
                                             "colored": ASSEMBLE_COLORED,
                                             "auto": 0}[mode]
        nnz = self.nnz()
        out = self._out(out, nnz)
        _check(load_library().fem_assemble_csr(self._h, _ptr(z), _ptr(out), flags, _stream()),
               "fem_assemble_csr")
        return out

    def spmv(self, vals: torch.Tensor, x, out=None) -> torch.Tensor:
        x = self._vec(x, "x")
        out = self._out(out)
        _check(load_library().fem_spmv(self._h, _ptr(vals), _ptr(x), _ptr(out), _stream()), "fem_spmv")
        return out

    def linearize(self, z) -> None:
        """Cache the tangent state at z for FEM_LINEARIZED HVPs (fem_linearize)."""
        z = self._vec(z, "z")
        _check(load_library().fem_linearize(self._h, _ptr(z), _stream()), "fem_linearize")

    def cg_solve(self, b, x0=None, z=None, vals=None, op: int = 0, rtol=1e-8, atol=0.0,
                 max_iter=100000, jacobi=False, check_every=1, raise_on_fail=True,
                 linearized=False):
        b = self._vec(b, "b")
        x = torch.zeros_like(b) if x0 is None else self._vec(x0, "x0").clone()
        zz = None if z is None else self._vec(z, "z")
        o = CgOpts(op, rtol, atol, max_iter, int(jacobi), check_every,
                   LINEARIZED if linearized else 0)
        rep = CgReport()
        st = load_library().fem_cg_solve(self._h, _ptr(zz), _ptr(vals), _ptr(b), _ptr(x),
                                         C.byref(o), C.byref(rep), _stream())
        info = {"status": st, "iters": rep.iters, "converged": bool(rep.converged),
                "res0": rep.res0, "res": rep.res}
        if raise_on_fail:
            _check(st, "fem_cg_solve")
        return x, info

    def minres_solve(self, b, x0=None, z=None, vals=None, op: int = 0, rtol=1e-8, atol=0.0,
                     max_iter=100000, check_every=1, raise_on_fail=True):
        """MINRES on the BC-applied operator (symmetric indefinite saddle points, f2)."""
        b = self._vec(b, "b")
        x = torch.zeros_like(b) if x0 is None else self._vec(x0, "x0").clone()
        zz = None if z is None else self._vec(z, "z")
        o = CgOpts(op, rtol, atol, max_iter, 0, check_every, 0)
        rep = CgReport()
        st = load_library().fem_minres_solve(self._h, _ptr(zz), _ptr(vals), _ptr(b), _ptr(x),
                                             C.byref(o), C.byref(rep), _stream())
        info = {"status": st, "iters": rep.iters, "converged": bool(rep.converged),
                "res0": rep.res0, "res": rep.res}
        if raise_on_fail:
            _check(st, "fem_minres_solve")
        return x, info

    def mean_stress(self, z) -> tuple:
        """(volume-averaged P as a dim x dim numpy array, |Omega|) — fem_mean_stress."""
        z = self._vec(z, "z")
        sig = (C.c_double * (self.dim * self.dim))()
        vol = C.c_double()
        _check(load_library().fem_mean_stress(self._h, _ptr(z), sig, C.byref(vol), _stream()),
               "fem_mean_stress")
        return np.array(sig[:], dtype=np.float64).reshape(self.dim, self.dim), vol.value

    def add_traction(self, facets, traction) -> None:
        """Psi -= int t . u over boundary facets (Line2 / Tri3); traction [n_facets][dim]
        (or one [dim] vector for all) — fem_add_traction."""
        f = torch.as_tensor(np.ascontiguousarray(facets, dtype=np.int32), device=self.device)
        t = np.asarray(traction, np.float64)
        if t.ndim == 1:
            t = np.tile(t, (len(f), 1))
        t = torch.as_tensor(np.ascontiguousarray(t), device=self.device)
        _check(load_library().fem_add_traction(self._h, len(f), _ptr(f), _ptr(t), _stream()),
               "fem_add_traction")

    def add_body_force(self, b) -> None:
        bb = (C.c_double * 3)(*([float(x) for x in b] + [0.0] * (3 - len(b))))
        _check(load_library().fem_add_body_force(self._h, bb, _stream()), "fem_add_body_force")

    def f_ext(self) -> torch.Tensor:
        out = torch.empty(self.n_u, dtype=torch.float64, device=self.device)
        _check(load_library().fem_get_fext(self._h, _ptr(out), _stream()), "fem_get_fext")
        return out

    # ---------------------------------------------------------------- multi-GPU halo
    def halo_size(self) -> int:
        n = C.c_int64()
        _check(load_library().fem_halo_size(self._h, C.byref(n)), "fem_halo_size")
        return n.value

    def halo_pack(self, y: torch.Tensor, send: Optional[torch.Tensor] = None) -> torch.Tensor:
        send = self._out(send, max(self.halo_size(), 1))
        _check(load_library().fem_halo_pack(self._h, _ptr(y), _ptr(send), _stream()), "fem_halo_pack")
        return send

    def halo_combine(self, y: torch.Tensor, recv: torch.Tensor) -> torch.Tensor:
        _check(load_library().fem_halo_combine(self._h, _ptr(y), _ptr(recv), _stream()),
               "fem_halo_combine")
        return y

    def newton_solve(self, z0, atol=1e-12, rtol=1e-10, max_iter=50, op=0, cg_rtol=1e-10,
                     cg_max_iter=100000, jacobi=False, check_every=1, raise_on_fail=True,
                     forcing=0.0):
        """forcing = 0: inner CG to cg_rtol at every step; in (0, 1]: Eisenstat-Walker
        forcing terms with gamma = forcing (fem.h fem_newton_opts, DESIGN reading R16)."""
        z = self._vec(z0, "z0").clone()
        o = NewtonOpts(atol, rtol, max_iter, CgOpts(op, cg_rtol, 0.0, cg_max_iter, int(jacobi),
                                                    check_every, 0), float(forcing))
        rep = NewtonReport()
        st = load_library().fem_newton_solve(self._h, _ptr(z), C.byref(o), C.byref(rep), _stream())
        info = {"status": st, "iters": rep.iters, "cg_iters": rep.cg_iters,
                "converged": bool(rep.converged), "res0": rep.res0, "res": rep.res}
        if raise_on_fail:
            _check(st, "fem_newton_solve")
        return z, info


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load_library().fem_nccl_unique_id(buf), "fem_nccl_unique_id")
    return buf.raw


def nccl_comm_init(uid: bytes, rank: int, size: int):
    comm = C.c_void_p()
    _check(load_library().fem_nccl_comm_init(C.create_string_buffer(uid, 128), rank, size,
                                             C.byref(comm)), "fem_nccl_comm_init")
    return comm.value


def nccl_comm_count(comm) -> int:
    n = C.c_int(0)
    _check(load_library().fem_nccl_comm_count(comm, C.byref(n)), "fem_nccl_comm_count")
    return n.value


def nccl_comm_destroy(comm) -> None:
    load_library().fem_nccl_comm_destroy(comm)


class VirtualWorkProblem:
    """Non-variational path (fem_vw_*): scalar advection-diffusion virtual
    work W(c, v) on a P1 mesh; residual r = grad_v W at v = 0, the non-symmetric JVP and
    GMRES.  Argument marshalling only."""

    def __init__(self, coords, conn, diffusivity, velocity, mass_coef=0.0, dirichlet_nodes=None,
                 dirichlet_vals=None, device="cuda"):
        lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("VirtualWorkProblem needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device)
        coords = np.ascontiguousarray(coords, np.float64)
        conn = np.ascontiguousarray(conn, np.int32)
        vel = np.ascontiguousarray(velocity, np.float64)
        dn = np.ascontiguousarray(np.zeros(0) if dirichlet_nodes is None else dirichlet_nodes, np.int32)
        dv = np.ascontiguousarray(np.zeros(0) if dirichlet_vals is None else dirichlet_vals, np.float64)
        self.n = coords.shape[0]
        self._keep = (coords, conn, vel, dn, dv)
        d = VwDesc(coords.shape[1], self.n, conn.shape[0], coords.ctypes.data, conn.ctypes.data,
                   diffusivity, vel.ctypes.data, mass_coef, len(dn),
                   dn.ctypes.data if len(dn) else None, dv.ctypes.data if len(dv) else None)
        h = C.c_void_p()
        _check(lib.fem_vw_create(C.byref(h), C.byref(d), _stream()), "fem_vw_create")
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            load_library().fem_vw_destroy(self._h)
            self._h = None

    def _vec(self, x):
        t = torch.as_tensor(x, dtype=torch.float64, device=self.device)
        if t.numel() != self.n:
            raise ValueError(f"expected {self.n} entries, got {t.numel()}")
        return t.contiguous()

    def apply_dirichlet(self, c):
        _check(load_library().fem_vw_apply_dirichlet(self._h, _ptr(c), _stream()), "fem_vw_apply_dirichlet")
        return c

    def residual(self, c, c_old=None, bc=False):
        c = self._vec(c)
        co = None if c_old is None else self._vec(c_old)
        r = torch.empty(self.n, dtype=torch.float64, device=self.device)
        _check(load_library().fem_vw_residual(self._h, _ptr(c), _ptr(co), _ptr(r),
                                              APPLY_BC if bc else 0, _stream()), "fem_vw_residual")
        return r

    def jvp(self, x, bc=False):
        x = self._vec(x)
        y = torch.empty(self.n, dtype=torch.float64, device=self.device)
        _check(load_library().fem_vw_jvp(self._h, _ptr(x), _ptr(y), APPLY_BC if bc else 0,
                                         _stream()), "fem_vw_jvp")
        return y

    def gmres_solve(self, b, x0=None, restart=30, max_iter=10000, rtol=1e-10, atol=0.0,
                    raise_on_fail=True):
        b = self._vec(b)
        x = torch.zeros_like(b) if x0 is None else self._vec(x0).clone()
        o = GmresOpts(restart, max_iter, rtol, atol)
        rep = CgReport()
        st = load_library().fem_vw_gmres_solve(self._h, _ptr(b), _ptr(x), C.byref(o), C.byref(rep),
                                               _stream())
        info = {"status": st, "iters": rep.iters, "converged": bool(rep.converged),
                "res0": rep.res0, "res": rep.res}
        if raise_on_fail:
            _check(st, "fem_vw_gmres_solve")
        return x, info
