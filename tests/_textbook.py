"""Textbook linear-elastic stiffness K = sum_e vol_e B_e^T D B_e (Voigt notation).

An independent routine for pinning the oracle (north_star: "the residual of linear
elasticity equals K.u").  It shares nothing with oracle/oracle.c: P1 gradients come
from inverting the barycentric matrix [[1 ... 1], [x_0 ... x_d]] with numpy, the
material enters through the plane-strain / 3D Voigt matrix D (standard references,
e.g. Zienkiewicz & Taylor vol. 1 ch. 4/6; Hughes ch. 2), and engineering shear
strains are used.  Dense, so only for small meshes.
"""
import math

import numpy as np


def barycentric_gradients(x):
    """x: [nen, d] vertex coords -> (grads [nen, d], volume)."""
    nen, d = x.shape
    M = np.vstack([np.ones(nen), x.T])        # [(d+1), nen]
    Minv = np.linalg.inv(M)                   # N(x) = Minv @ [1; x]
    return Minv[:, 1:], abs(np.linalg.det(M)) / math.factorial(d)


def voigt_D(d, lam, mu):
    if d == 2:   # plane strain (reading C2)
        return np.array([[lam + 2 * mu, lam, 0.0], [lam, lam + 2 * mu, 0.0], [0.0, 0.0, mu]])
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2 * mu
    D[np.arange(3, 6), np.arange(3, 6)] = mu
    return D


def voigt_B(grads):
    nen, d = grads.shape
    if d == 2:
        B = np.zeros((3, 2 * nen))
        for a in range(nen):
            gx, gy = grads[a]
            B[0, 2 * a] = gx
            B[1, 2 * a + 1] = gy
            B[2, 2 * a] = gy
            B[2, 2 * a + 1] = gx
        return B
    B = np.zeros((6, 3 * nen))
    for a in range(nen):
        gx, gy, gz = grads[a]
        c = 3 * a
        B[0, c] = gx
        B[1, c + 1] = gy
        B[2, c + 2] = gz
        B[3, c + 1], B[3, c + 2] = gz, gy
        B[4, c], B[4, c + 2] = gz, gx
        B[5, c], B[5, c + 1] = gy, gx
    return B


def stiffness(mesh):
    d = mesh.dim
    N = mesh.n_u
    K = np.zeros((N, N))
    for e in range(mesh.n_elems):
        nodes = mesh.conn[e]
        if mesh.phase is not None:
            lam, mu = mesh.lambda_tab[mesh.phase[e]], mesh.mu_tab[mesh.phase[e]]
        else:
            lam, mu = mesh.lam, mesh.mu
        g, vol = barycentric_gradients(mesh.coords[nodes])
        B = voigt_B(g)
        Ke = vol * B.T @ voigt_D(d, lam, mu) @ B
        dofs = (nodes[:, None] * d + np.arange(d)).ravel()
        K[np.ix_(dofs, dofs)] += Ke
    return K


def strain_energy_density(H, lam, mu):
    """0.5 eps^T D eps with engineering shear, eps = sym(H) in Voigt order."""
    d = H.shape[0]
    e = 0.5 * (H + H.T)
    if d == 2:
        v = np.array([e[0, 0], e[1, 1], 2 * e[0, 1]])
    else:
        v = np.array([e[0, 0], e[1, 1], e[2, 2], 2 * e[1, 2], 2 * e[0, 2], 2 * e[0, 1]])
    return 0.5 * v @ voigt_D(d, lam, mu) @ v


def constraint_matrix(mesh):
    """B = dg/du for g_k = u[s_k] - u[m_k] - b_k (App. B)."""
    B = np.zeros((mesh.n_mpc, mesh.n_u))
    B[np.arange(mesh.n_mpc), mesh.mpc_slave] += 1.0
    B[np.arange(mesh.n_mpc), mesh.mpc_master] -= 1.0
    return B
