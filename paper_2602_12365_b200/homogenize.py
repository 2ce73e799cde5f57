"""Periodic homogenization driver (§6.2.2).

For each unit macroscopic strain in Voigt notation the periodic Lagrangian
L(u, lambda) = Psi(u) + lambda . g(u) is solved to stationarity with the
library's Newton iteration, whose inner solves are MINRES on the indefinite saddle-point
operator [[K, B^T], [B, 0]] (fem_newton_solve -> fem_minres_solve, CG does not apply).  The
macroscopic stress is the volume average of the microscopic stress (fem_mean_stress,
P:530-531).  For a linear-elastic RVE sigma_hom is linear in the macro strain, so the
columns sigma_hom(e_j) are exactly the Jacobian jax.jacfwd(solve) of the paper's listing
(P:536-543); reading R5.

Argument marshalling only: every step runs in libfem.so.  `make_mesh(eps_hat)` returns the
RVE mesh with its periodic constraint offsets b = eps_hat (X_s - X_m) for the given macro
strain (the constraints are set up by the caller, e.g. fem_inputs.periodic_mpc).
"""
from __future__ import annotations

import numpy as np
import torch

from . import fem


def voigt_unit_strains(dim: int):
    """Unit Voigt strains with engineering shear: 2D [xx, yy, xy], 3D [xx, yy, zz, yz, xz, xy]."""
    if dim == 2:
        pairs = [(0, 0), (1, 1), (0, 1)]
    else:
        pairs = [(0, 0), (1, 1), (2, 2), (1, 2), (0, 2), (0, 1)]
    out = []
    for i, j in pairs:
        e = np.zeros((dim, dim))
        if i == j:
            e[i, i] = 1.0
        else:
            e[i, j] = e[j, i] = 0.5   # gamma_ij = 2 eps_ij = 1
        out.append(e)
    return pairs, out


def to_voigt(sig: np.ndarray, pairs) -> np.ndarray:
    return np.array([0.5 * (sig[i, j] + sig[j, i]) for i, j in pairs])


def solve_rve(mesh, rtol: float = 1e-12, atol: float = 1e-14, max_iter: int = 20,
              inner_rtol: float = 1e-13, inner_max_iter: int = 200000):
    """Stationary point of the periodic Lagrangian on `mesh` (Newton + MINRES); returns
    (z, newton report, Problem)."""
    prob = fem.Problem(mesh)
    z0 = torch.zeros(mesh.n_total, dtype=torch.float64, device="cuda")
    prob.apply_dirichlet(z0)
    z, info = prob.newton_solve(z0, atol=atol, rtol=rtol, max_iter=max_iter, op=0,
                                cg_rtol=inner_rtol, cg_max_iter=inner_max_iter, check_every=16)
    return z, info, prob


def homogenized_stiffness(make_mesh, dim: int, **kw):
    """C_hom (Voigt, engineering shear): column j = volume-averaged stress of the RVE solved
    at unit macro strain e_j.  Returns (C_hom, per-case reports)."""
    pairs, strains = voigt_unit_strains(dim)
    cols, reports = [], []
    for e in strains:
        mesh = make_mesh(e)
        z, info, prob = solve_rve(mesh, **kw)
        sig, vol = prob.mean_stress(z)
        cols.append(to_voigt(sig, pairs))
        reports.append({**info, "volume": vol})
    return np.stack(cols, axis=1), reports
