/*
 * oracle.c — plain, slow, single-threaded CPU oracle for the hot path of
 * arXiv 2602.12365 ("tatva"): energy, residual, HVP, sparsity pattern,
 * distance-2 greedy coloring, Alg. 2 colored assembly, SpMV, CG, Newton.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2602_12365_b200/csrc).
 *
 * How it computes:
 *   * The element energy E_e(u_e) = vol_e * psi(H(u_e)) is the only physics
 *     formula here (Eq. 2; Alg. 1).  The residual,
 *     the HVP and the element Hessian are its exact derivatives, taken by
 *     forward-mode (hyper-)dual numbers seeded on the element's nodal DOFs
 *     (Eq. 1: r = grad Psi, K = hess Psi).  The oracle therefore
 *     never contains the hand-derived first Piola stress or tangent modulus that
 *     the GPU kernels use.
 *   * Sums over elements run in ascending element order; global scalar sums are
 *     Neumaier-compensated (reading C10).  Compiled with -O2 -ffp-contract=off.
 *
 * Parity pins: every function below is pinned in tests/test_oracle_*.py against
 * closed forms, brute force, textbook routines or library routines (DESIGN.md §3
 * table).  No function is "parity unpinned".
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, E_ARG = 1, E_DEGENERATE = 2, E_INVERTED = 3, E_NONFINITE = 4, E_BREAKDOWN = 5,
       E_NOTCONV = 6, E_OOM = 8 };

/* ------------------------------------------------------------------ hyper-dual numbers
 * x = a + b e1 + c e2 + d e1 e2 with e1^2 = e2^2 = 0 (Fike & Alonso).  The e1 part of
 * f(x + e1 s) is the directional derivative f'(x) s; the e1e2 part of
 * f(x + e1 s + e2 t) is s^T f''(x) t, exactly (no truncation).  psi needs only
 * +, -, *, / (by a real constant) and log.                                           */
typedef struct { double a, b, c, d; } hd;

static hd hd_const(double a) { hd r = {a, 0.0, 0.0, 0.0}; return r; }
static hd hd_add(hd x, hd y) { hd r = {x.a + y.a, x.b + y.b, x.c + y.c, x.d + y.d}; return r; }
static hd hd_sub(hd x, hd y) { hd r = {x.a - y.a, x.b - y.b, x.c - y.c, x.d - y.d}; return r; }
static hd hd_mul(hd x, hd y) {
  hd r;
  r.a = x.a * y.a;
  r.b = x.a * y.b + x.b * y.a;
  r.c = x.a * y.c + x.c * y.a;
  r.d = x.a * y.d + x.b * y.c + x.c * y.b + x.d * y.a;
  return r;
}
static hd hd_scale(hd x, double s) { hd r = {x.a * s, x.b * s, x.c * s, x.d * s}; return r; }
/* ln(a + b e1 + c e2 + d e1e2) = ln a + (b/a) e1 + (c/a) e2 + (d/a - b c / a^2) e1e2 */
static hd hd_log(hd x) {
  hd r;
  r.a = log(x.a);
  r.b = x.b / x.a;
  r.c = x.c / x.a;
  r.d = x.d / x.a - x.b * x.c / (x.a * x.a);
  return r;
}

/* Neumaier compensated accumulator (reading C10). */
typedef struct { double s, c; } ksum;
static void ks_add(ksum *k, double x) {
  double t = k->s + x;
  if (fabs(k->s) >= fabs(x)) k->c += (k->s - t) + x;
  else k->c += (x - t) + k->s;
  k->s = t;
}
static double ks_val(const ksum *k) { return k->s + k->c; }

/* ------------------------------------------------------------------ energy density psi
 * Linear elastic (listing `strain_energy_density`, plane strain in
 * 2D, reading C2):  eps = (H + H^T)/2,  sig = 2 mu eps + lambda tr(eps) I,
 * psi = 0.5 sig : eps.
 * Compressible neo-Hookean (PAPER.md P:418-430 elides the body, "... # do stuff";
 * reading C1 = SPEC S:643):  F = I + H,  C = F^T F (as in the listing),
 * I1 = tr C,  J = det F,  psi = mu/2 (I1 - d - 2 ln J) + lambda/2 (ln J)^2.
 * Returns E_INVERTED when J <= 0.                                        */
static int psi_hd(int dim, int material, double lam, double mu, hd H[3][3], hd *out) {
  int i, j, k;
  if (material == 0) {
    hd eps[3][3], sig[3][3], tr = hd_const(0.0), s = hd_const(0.0);
    for (i = 0; i < dim; ++i)
      for (j = 0; j < dim; ++j) eps[i][j] = hd_scale(hd_add(H[i][j], H[j][i]), 0.5);
    for (i = 0; i < dim; ++i) tr = hd_add(tr, eps[i][i]);
    for (i = 0; i < dim; ++i)
      for (j = 0; j < dim; ++j) {
        sig[i][j] = hd_scale(eps[i][j], 2.0 * mu);
        if (i == j) sig[i][j] = hd_add(sig[i][j], hd_scale(tr, lam));
      }
    for (i = 0; i < dim; ++i)
      for (j = 0; j < dim; ++j) s = hd_add(s, hd_mul(sig[i][j], eps[i][j]));
    *out = hd_scale(s, 0.5);
    return OK;
  } else {
    hd F[3][3], C[3][3], I1 = hd_const(0.0), J, lnJ, t;
    for (i = 0; i < dim; ++i)
      for (j = 0; j < dim; ++j) F[i][j] = (i == j) ? hd_add(H[i][j], hd_const(1.0)) : H[i][j];
    for (i = 0; i < dim; ++i)
      for (j = 0; j < dim; ++j) {
        C[i][j] = hd_const(0.0);
        for (k = 0; k < dim; ++k) C[i][j] = hd_add(C[i][j], hd_mul(F[k][i], F[k][j]));
      }
    for (i = 0; i < dim; ++i) I1 = hd_add(I1, C[i][i]);
    if (dim == 2) {
      J = hd_sub(hd_mul(F[0][0], F[1][1]), hd_mul(F[0][1], F[1][0]));
    } else { /* cofactor expansion along the first row */
      hd c0 = hd_sub(hd_mul(F[1][1], F[2][2]), hd_mul(F[1][2], F[2][1]));
      hd c1 = hd_sub(hd_mul(F[1][2], F[2][0]), hd_mul(F[1][0], F[2][2]));
      hd c2 = hd_sub(hd_mul(F[1][0], F[2][1]), hd_mul(F[1][1], F[2][0]));
      J = hd_add(hd_add(hd_mul(F[0][0], c0), hd_mul(F[0][1], c1)), hd_mul(F[0][2], c2));
    }
    if (!(J.a > 0.0)) return E_INVERTED;
    lnJ = hd_log(J);
    t = hd_sub(hd_sub(I1, hd_const((double)dim)), hd_scale(lnJ, 2.0));
    *out = hd_add(hd_scale(t, 0.5 * mu), hd_scale(hd_mul(lnJ, lnJ), 0.5 * lam));
    return OK;
  }
}

/* ------------------------------------------------------------------ element geometry
 * P1 simplex, one-point rule (reading C4): x(xi) = x0 + J xi with J = [x1-x0 | ... ]
 * (columns are edge vectors).  grad N_a = J^{-T} grad_xi N_a, so for a >= 1 G_a is row
 * a-1 of J^{-1}, and G_0 = -sum_{a>=1} G_a (reference gradients SPEC S:146).
 * vol = w * det J with w = 1/2 (Tri3), 1/6 (Tet4) (Eq. 2 "w_q det J").
 * det J <= eps_det = 1e-14 * (bbox diagonal)^d -> DegenerateElement (reading C20).   */
static int elem_geometry(const fem_ref_mesh *m, int64_t e, double G[4][3], double *vol) {
  int d = m->dim, nen = d + 1, a, i, j;
  double x[4][3], Jm[3][3], inv[3][3], det, lo[3], hi[3], diag2 = 0.0, epsd;
  for (a = 0; a < nen; ++a) {
    int64_t n = m->conn[e * nen + a];
    for (i = 0; i < d; ++i) x[a][i] = m->coords[n * d + i];
  }
  for (i = 0; i < d; ++i) {
    lo[i] = hi[i] = x[0][i];
    for (a = 1; a < nen; ++a) {
      if (x[a][i] < lo[i]) lo[i] = x[a][i];
      if (x[a][i] > hi[i]) hi[i] = x[a][i];
    }
    diag2 += (hi[i] - lo[i]) * (hi[i] - lo[i]);
  }
  for (i = 0; i < d; ++i)
    for (j = 0; j < d; ++j) Jm[i][j] = x[j + 1][i] - x[0][i];
  if (d == 2) {
    det = Jm[0][0] * Jm[1][1] - Jm[0][1] * Jm[1][0];
    epsd = 1e-14 * diag2;
    if (!(det > epsd)) return E_DEGENERATE;
    inv[0][0] = Jm[1][1] / det;  inv[0][1] = -Jm[0][1] / det;
    inv[1][0] = -Jm[1][0] / det; inv[1][1] = Jm[0][0] / det;
    *vol = det / 2.0;
  } else {
    double cof[3][3];
    cof[0][0] = Jm[1][1] * Jm[2][2] - Jm[1][2] * Jm[2][1];
    cof[0][1] = Jm[1][2] * Jm[2][0] - Jm[1][0] * Jm[2][2];
    cof[0][2] = Jm[1][0] * Jm[2][1] - Jm[1][1] * Jm[2][0];
    cof[1][0] = Jm[0][2] * Jm[2][1] - Jm[0][1] * Jm[2][2];
    cof[1][1] = Jm[0][0] * Jm[2][2] - Jm[0][2] * Jm[2][0];
    cof[1][2] = Jm[0][1] * Jm[2][0] - Jm[0][0] * Jm[2][1];
    cof[2][0] = Jm[0][1] * Jm[1][2] - Jm[0][2] * Jm[1][1];
    cof[2][1] = Jm[0][2] * Jm[1][0] - Jm[0][0] * Jm[1][2];
    cof[2][2] = Jm[0][0] * Jm[1][1] - Jm[0][1] * Jm[1][0];
    det = Jm[0][0] * cof[0][0] + Jm[0][1] * cof[0][1] + Jm[0][2] * cof[0][2];
    epsd = 1e-14 * diag2 * sqrt(diag2);
    if (!(det > epsd)) return E_DEGENERATE;
    /* J^{-1} = adj(J)/det = cof^T / det */
    for (i = 0; i < 3; ++i)
      for (j = 0; j < 3; ++j) inv[i][j] = cof[j][i] / det;
    *vol = det / 6.0;
  }
  for (i = 0; i < d; ++i) G[0][i] = 0.0;
  for (a = 1; a < nen; ++a)
    for (i = 0; i < d; ++i) {
      G[a][i] = inv[a - 1][i];
      G[0][i] -= inv[a - 1][i];
    }
  return OK;
}

static void elem_material(const fem_ref_mesh *m, int64_t e, double *lam, double *mu) {
  if (m->phase) {
    *lam = m->lambda_tab[m->phase[e]];
    *mu = m->mu_tab[m->phase[e]];
  } else {
    *lam = m->lambda;
    *mu = m->mu;
  }
}

/* Element energy E_e = vol * psi(H), H_ij = sum_a u_{a,i} G_{a,j}
 * (Alg. 1 P:129-136 "field gradients", "integrate").                       */
static int elem_energy_hd(const fem_ref_mesh *m, int64_t e, double G[4][3], double vol,
                          hd ue[4][3], hd *out) {
  int d = m->dim, nen = d + 1, a, i, j, st;
  double lam, mu;
  hd H[3][3], p;
  elem_material(m, e, &lam, &mu);
  for (i = 0; i < d; ++i)
    for (j = 0; j < d; ++j) {
      H[i][j] = hd_const(0.0);
      for (a = 0; a < nen; ++a) H[i][j] = hd_add(H[i][j], hd_scale(ue[a][i], G[a][j]));
    }
  st = psi_hd(d, m->material, lam, mu, H, &p);
  if (st) return st;
  *out = hd_scale(p, vol);
  return OK;
}

static int64_t n_u(const fem_ref_mesh *m) { return m->n_nodes * m->dim; }
static int64_t n_tot(const fem_ref_mesh *m) { return n_u(m) + m->n_mpc; }

static unsigned char *dirichlet_mask(const fem_ref_mesh *m) {
  unsigned char *mask = (unsigned char *)calloc((size_t)n_tot(m) + 1, 1);
  int64_t k;
  if (!mask) return NULL;
  for (k = 0; k < m->n_dirichlet; ++k) mask[m->dirichlet_dofs[k]] = 1;
  return mask;
}

static int check_finite(const double *x, int64_t n) {
  int64_t i;
  for (i = 0; i < n; ++i)
    if (!isfinite(x[i])) return E_NONFINITE;
  return OK;
}

/* ------------------------------------------------------------------ geometry export */
int fem_ref_geometry(const fem_ref_mesh *m, double *G, double *vol) {
  int64_t e;
  int d = m->dim, nen = d + 1, a, i, st;
  double g[4][3], v;
  for (e = 0; e < m->n_elems; ++e) {
    st = elem_geometry(m, e, g, &v);
    if (st) return st;
    for (a = 0; a < nen; ++a)
      for (i = 0; i < d; ++i) G[(e * nen + a) * d + i] = g[a][i];
    vol[e] = v;
  }
  return OK;
}

/* ------------------------------------------------------------------ O-energy
 * Psi_h = sum_e vol_e psi(H_e) (Eq. 2, Alg. 1), + lambda . g(u) (Lagrangian,
 * P:497-498), - f_ext . u.  Ascending element order, Neumaier-compensated.           */
int fem_ref_energy(const fem_ref_mesh *m, const double *z, double *energy) {
  int d = m->dim, nen = d + 1, a, i, st;
  int64_t e, k, nu = n_u(m);
  ksum acc = {0.0, 0.0};
  double G[4][3], vol;
  hd ue[4][3], Ee;
  for (e = 0; e < m->n_elems; ++e) {
    st = elem_geometry(m, e, G, &vol);
    if (st) return st;
    for (a = 0; a < nen; ++a)
      for (i = 0; i < d; ++i) ue[a][i] = hd_const(z[(int64_t)m->conn[e * nen + a] * d + i]);
    st = elem_energy_hd(m, e, G, vol, ue, &Ee);
    if (st) return st;
    ks_add(&acc, Ee.a);
  }
  for (k = 0; k < m->n_mpc; ++k)
    ks_add(&acc, z[nu + k] * (z[m->mpc_slave[k]] - z[m->mpc_master[k]] - m->mpc_offset[k]));
  if (m->f_ext)
    for (k = 0; k < nu; ++k) ks_add(&acc, -m->f_ext[k] * z[k]);
  *energy = ks_val(&acc);
  return isfinite(*energy) ? OK : E_NONFINITE;
}

/* Gradient (seed s2 = NULL) or Hessian-vector product (seed s2 = w) of the element
 * energy with respect to each element DOF (a,i), by seeding u_e + e1 e_(a,i) [+ e2 w_e]:
 * out[a][i] = dE_e/du_(a,i)   (dual part)      — reverse-mode residual
 * out[a][i] = (K_e w_e)_(a,i) (e1e2 part)      — forward-over-reverse JVP, Eq. 3.    */
static int elem_derivative(const fem_ref_mesh *m, int64_t e, const double *z, const double *w,
                           double out[4][3]) {
  int d = m->dim, nen = d + 1, a, i, b, k, st;
  double G[4][3], vol;
  hd ue[4][3], Ee;
  st = elem_geometry(m, e, G, &vol);
  if (st) return st;
  for (a = 0; a < nen; ++a)
    for (i = 0; i < d; ++i) {
      for (b = 0; b < nen; ++b)
        for (k = 0; k < d; ++k) {
          int64_t dof = (int64_t)m->conn[e * nen + b] * d + k;
          ue[b][k] = hd_const(z[dof]);
          if (w) ue[b][k].c = w[dof];
        }
      ue[a][i].b = 1.0;
      st = elem_energy_hd(m, e, G, vol, ue, &Ee);
      if (st) return st;
      out[a][i] = w ? Ee.d : Ee.b;
    }
  return OK;
}

/* ------------------------------------------------------------------ O-residual
 * r = grad L(z): element gradients scattered in ascending element order; then the
 * multiplier terms r_u += B^T lambda, r_lambda = B u - b (App. B);
 * r_u -= f_ext; with FEM_REF_APPLY_BC r[D] = 0 (condensation realised on full-length
 * vectors, reading C12).                                                  */
int fem_ref_residual(const fem_ref_mesh *m, const double *z, double *r, unsigned flags) {
  int d = m->dim, nen = d + 1, a, i, st;
  int64_t e, k, nu = n_u(m), N = n_tot(m);
  double f[4][3];
  memset(r, 0, sizeof(double) * (size_t)N);
  for (e = 0; e < m->n_elems; ++e) {
    st = elem_derivative(m, e, z, NULL, f);
    if (st) return st;
    for (a = 0; a < nen; ++a)
      for (i = 0; i < d; ++i) r[(int64_t)m->conn[e * nen + a] * d + i] += f[a][i];
  }
  for (k = 0; k < m->n_mpc; ++k) {
    r[m->mpc_slave[k]] += z[nu + k];
    r[m->mpc_master[k]] -= z[nu + k];
    r[nu + k] = z[m->mpc_slave[k]] - z[m->mpc_master[k]] - m->mpc_offset[k];
  }
  if (m->f_ext)
    for (k = 0; k < nu; ++k) r[k] -= m->f_ext[k];
  if (flags & FEM_REF_APPLY_BC)
    for (k = 0; k < m->n_dirichlet; ++k) r[m->dirichlet_dofs[k]] = 0.0;
  return check_finite(r, N);
}

/* ------------------------------------------------------------------ O-hvp
 * y = K(z) v (Eq. 3), K the Hessian of the Lagrangian:
 * y_u = K_uu v_u + B^T v_lambda, y_lambda = B v_u.  With FEM_REF_APPLY_BC the masked
 * operator y = P_f K P_f v + P_D v (reading C12).                                     */
int fem_ref_hvp(const fem_ref_mesh *m, const double *z, const double *v, double *y,
                unsigned flags) {
  int d = m->dim, nen = d + 1, a, i, st;
  int64_t e, k, nu = n_u(m), N = n_tot(m);
  double f[4][3], *w = (double *)malloc(sizeof(double) * (size_t)N);
  if (!w) return E_OOM;
  memcpy(w, v, sizeof(double) * (size_t)N);
  if (flags & FEM_REF_APPLY_BC)
    for (k = 0; k < m->n_dirichlet; ++k) w[m->dirichlet_dofs[k]] = 0.0;
  memset(y, 0, sizeof(double) * (size_t)N);
  for (e = 0; e < m->n_elems; ++e) {
    st = elem_derivative(m, e, z, w, f);
    if (st) { free(w); return st; }
    for (a = 0; a < nen; ++a)
      for (i = 0; i < d; ++i) y[(int64_t)m->conn[e * nen + a] * d + i] += f[a][i];
  }
  for (k = 0; k < m->n_mpc; ++k) {
    y[m->mpc_slave[k]] += w[nu + k];
    y[m->mpc_master[k]] -= w[nu + k];
    y[nu + k] = w[m->mpc_slave[k]] - w[m->mpc_master[k]];
  }
  if (flags & FEM_REF_APPLY_BC)
    for (k = 0; k < m->n_dirichlet; ++k) y[m->dirichlet_dofs[k]] = v[m->dirichlet_dofs[k]];
  free(w);
  return check_finite(y, N);
}

/* ------------------------------------------------------------------ O-dense
 * H[:, j] = hvp(z, e_j) — the dense Hessian the paper avoids.         */
int fem_ref_dense_hessian(const fem_ref_mesh *m, const double *z, double *H, unsigned flags) {
  int64_t N = n_tot(m), j, i;
  int st = OK;
  double *ej = (double *)calloc((size_t)N, sizeof(double));
  double *col = (double *)malloc(sizeof(double) * (size_t)N);
  if (!ej || !col) { free(ej); free(col); return E_OOM; }
  for (j = 0; j < N && st == OK; ++j) {
    ej[j] = 1.0;
    st = fem_ref_hvp(m, z, ej, col, flags);
    ej[j] = 0.0;
    for (i = 0; i < N; ++i) H[i * N + j] = col[i];
  }
  free(ej);
  free(col);
  return st;
}

/* node -> incident elements (ascending element order), for the row-sampled checks */
static int build_incidence(const fem_ref_mesh *m, int64_t **ptr_out, int64_t **elem_out) {
  int nen = m->dim + 1, a;
  int64_t e, n, *ptr = (int64_t *)calloc((size_t)m->n_nodes + 1, sizeof(int64_t)), *fill, *el;
  if (!ptr) return E_OOM;
  for (e = 0; e < m->n_elems; ++e)
    for (a = 0; a < nen; ++a) ptr[m->conn[e * nen + a] + 1]++;
  for (n = 0; n < m->n_nodes; ++n) ptr[n + 1] += ptr[n];
  el = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ptr[m->n_nodes] + 1));
  fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m->n_nodes + 1));
  if (!el || !fill) { free(ptr); free(el); free(fill); return E_OOM; }
  memcpy(fill, ptr, sizeof(int64_t) * (size_t)m->n_nodes);
  for (e = 0; e < m->n_elems; ++e)
    for (a = 0; a < nen; ++a) el[fill[m->conn[e * nen + a]]++] = e;
  free(fill);
  *ptr_out = ptr;
  *elem_out = el;
  return OK;
}

/* Row-sampled residual / HVP: the same sums as fem_ref_residual / fem_ref_hvp, for the
 * requested rows only, from the incident elements in ascending element order.  Used for
 * parity at the full BASELINE sizes where the whole-mesh oracle is too slow.          */
static int rows_common(const fem_ref_mesh *m, const double *z, const double *v, int64_t n_rows,
                       const int64_t *rows, double *out, unsigned flags) {
  int d = m->dim, nen = d + 1, a, i, st = OK;
  int64_t *ptr = NULL, *el = NULL, q, t, k, nu = n_u(m);
  unsigned char *mask = dirichlet_mask(m);
  double f[4][3], *w = NULL;
  if (!mask) return E_OOM;
  st = build_incidence(m, &ptr, &el);
  if (st) { free(mask); return st; }
  if (v) {
    w = (double *)malloc(sizeof(double) * (size_t)n_tot(m));
    if (!w) { free(mask); free(ptr); free(el); return E_OOM; }
    memcpy(w, v, sizeof(double) * (size_t)n_tot(m));
    if (flags & FEM_REF_APPLY_BC)
      for (k = 0; k < m->n_dirichlet; ++k) w[m->dirichlet_dofs[k]] = 0.0;
  }
  for (q = 0; q < n_rows && st == OK; ++q) {
    int64_t row = rows[q];
    double acc = 0.0;
    if (row < nu) {
      int64_t node = row / d;
      int comp = (int)(row % d);
      for (t = ptr[node]; t < ptr[node + 1]; ++t) {
        int64_t e = el[t];
        st = elem_derivative(m, e, z, w, f);
        if (st) break;
        for (a = 0; a < nen; ++a)
          if (m->conn[e * nen + a] == node) acc += f[a][comp];
      }
      for (k = 0; k < m->n_mpc; ++k) {
        double lk = v ? w[nu + k] : z[nu + k];
        if (m->mpc_slave[k] == row) acc += lk;
        if (m->mpc_master[k] == row) acc -= lk;
      }
      if (!v && m->f_ext) acc -= m->f_ext[row];
    } else {
      k = row - nu;
      acc = v ? (w[m->mpc_slave[k]] - w[m->mpc_master[k]])
              : (z[m->mpc_slave[k]] - z[m->mpc_master[k]] - m->mpc_offset[k]);
    }
    if ((flags & FEM_REF_APPLY_BC) && mask[row]) acc = v ? v[row] : 0.0;
    out[q] = acc;
    (void)i;
  }
  free(mask); free(ptr); free(el); free(w);
  return st;
}

int fem_ref_residual_rows(const fem_ref_mesh *m, const double *z, int64_t n_rows,
                          const int64_t *rows, double *out, unsigned flags) {
  return rows_common(m, z, NULL, n_rows, rows, out, flags);
}

int fem_ref_hvp_rows(const fem_ref_mesh *m, const double *z, const double *v, int64_t n_rows,
                     const int64_t *rows, double *out, unsigned flags) {
  return rows_common(m, z, v, n_rows, rows, out, flags);
}

/* ------------------------------------------------------------------ O-pattern
 * (i, j) present iff DOFs i and j belong to nodes that share an element, i = j
 * included ("construct the sparsity pattern ... using mesh
 * connectivity"; App. B).  Full m x m node blocks.  With
 * multipliers: the union [[K, B^T], [B, 0]] (App. B), B_{k,s_k} and
 * B_{k,m_k} nonzero, empty multiplier-multiplier block.
 * Columns ascending in each row.  col_idx == NULL: only row_ptr is written.          */
static int cmp_i64(const void *x, const void *y) {
  int64_t a = *(const int64_t *)x, b = *(const int64_t *)y;
  return (a > b) - (a < b);
}

int fem_ref_sparsity(const fem_ref_mesh *m, int64_t *row_ptr, int32_t *col_idx) {
  int d = m->dim, nen = d + 1, a, b, c, c2;
  int64_t e, n, k, t, nu = n_u(m), N = n_tot(m), row;
  int64_t *cnt = (int64_t *)calloc((size_t)m->n_nodes + 1, sizeof(int64_t));
  int64_t *nptr, *nb, *fill, *nuniq;
  if (!cnt) return E_OOM;
  /* node neighbour lists: every node of every element containing n (with repeats) */
  for (e = 0; e < m->n_elems; ++e)
    for (a = 0; a < nen; ++a) cnt[m->conn[e * nen + a] + 1] += nen;
  nptr = cnt;
  for (n = 0; n < m->n_nodes; ++n) nptr[n + 1] += nptr[n];
  nb = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nptr[m->n_nodes] + 1));
  fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m->n_nodes + 1));
  nuniq = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m->n_nodes + 1));
  if (!nb || !fill || !nuniq) { free(cnt); free(nb); free(fill); free(nuniq); return E_OOM; }
  memcpy(fill, nptr, sizeof(int64_t) * (size_t)m->n_nodes);
  for (e = 0; e < m->n_elems; ++e)
    for (a = 0; a < nen; ++a)
      for (b = 0; b < nen; ++b) nb[fill[m->conn[e * nen + a]]++] = m->conn[e * nen + b];
  for (n = 0; n < m->n_nodes; ++n) { /* sort + unique in place */
    int64_t lo = nptr[n], hi = nptr[n + 1], u = lo;
    qsort(nb + lo, (size_t)(hi - lo), sizeof(int64_t), cmp_i64);
    for (t = lo; t < hi; ++t)
      if (t == lo || nb[t] != nb[t - 1]) nb[u++] = nb[t];
    nuniq[n] = u - lo;
  }
  /* row lengths */
  row_ptr[0] = 0;
  for (row = 0; row < N; ++row) {
    int64_t len;
    if (row < nu) {
      len = nuniq[row / d] * d;
      for (k = 0; k < m->n_mpc; ++k)
        len += (m->mpc_slave[k] == row) + (m->mpc_master[k] == row);
    } else {
      len = 2;
    }
    row_ptr[row + 1] = row_ptr[row] + len;
  }
  if (col_idx) {
    for (row = 0; row < N; ++row) {
      int64_t p = row_ptr[row];
      if (row < nu) {
        n = row / d;
        for (t = nptr[n]; t < nptr[n] + nuniq[n]; ++t)
          for (c2 = 0; c2 < d; ++c2) col_idx[p++] = (int32_t)(nb[t] * d + c2);
        for (k = 0; k < m->n_mpc; ++k)
          if (m->mpc_slave[k] == row || m->mpc_master[k] == row) col_idx[p++] = (int32_t)(nu + k);
      } else {
        int64_t s = m->mpc_slave[row - nu], ms = m->mpc_master[row - nu];
        col_idx[p++] = (int32_t)(s < ms ? s : ms);
        col_idx[p++] = (int32_t)(s < ms ? ms : s);
      }
    }
  }
  (void)c;
  free(cnt); free(nb); free(fill); free(nuniq);
  return OK;
}

/* ------------------------------------------------------------------ O-color
 * Distance-2 greedy coloring of the columns (App. A; §2.2; reading C8/C9):
 * columns visited in ascending index; column j gets the smallest color >= 0 not used by
 * any column j' < j that shares a row with j.  Rows of column j are
 * taken from the explicit transpose, so no symmetry is assumed.                      */
int fem_ref_color(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, int32_t *colors,
                  int32_t *n_colors) {
  int64_t nnz = row_ptr[n], i, j, p, q;
  int64_t *cptr = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t)), *cfill;
  int64_t *crow = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nnz + 1));
  int64_t *forbid = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  int32_t maxc = -1;
  if (!cptr || !crow || !forbid) { free(cptr); free(crow); free(forbid); return E_OOM; }
  for (p = 0; p < nnz; ++p) cptr[col_idx[p] + 1]++;
  for (j = 0; j < n; ++j) cptr[j + 1] += cptr[j];
  cfill = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  if (!cfill) { free(cptr); free(crow); free(forbid); return E_OOM; }
  memcpy(cfill, cptr, sizeof(int64_t) * (size_t)n);
  for (i = 0; i < n; ++i)
    for (p = row_ptr[i]; p < row_ptr[i + 1]; ++p) crow[cfill[col_idx[p]]++] = i;
  for (j = 0; j <= n; ++j) forbid[j] = -1;
  for (j = 0; j < n; ++j) {
    int32_t c = 0;
    for (p = cptr[j]; p < cptr[j + 1]; ++p) {
      int64_t r = crow[p];
      for (q = row_ptr[r]; q < row_ptr[r + 1]; ++q)
        if (col_idx[q] < j) forbid[colors[col_idx[q]]] = j;
    }
    while (forbid[c] == j) ++c;
    colors[j] = c;
    if (c > maxc) maxc = c;
  }
  *n_colors = maxc + 1;
  free(cptr); free(crow); free(forbid); free(cfill);
  return OK;
}

/* ------------------------------------------------------------------ O-alg2
 * Alg. 2 literally: for each color c, seed e_j = [color_j == c], compute
 * y = JVP of the residual along e (the HVP, with the same BC semantics), store y as
 * column c of J_comp [N x C]; then K_ij = J_comp[i, color[j]] over the pattern.      */
int fem_ref_assemble_alg2(const fem_ref_mesh *m, const double *z, const int64_t *row_ptr,
                          const int32_t *col_idx, const int32_t *colors, int32_t n_colors,
                          double *vals, unsigned flags) {
  int64_t N = n_tot(m), i, j, p;
  int32_t c;
  int st = OK;
  double *Jc = (double *)malloc(sizeof(double) * (size_t)N * (size_t)n_colors);
  double *e = (double *)malloc(sizeof(double) * (size_t)N);
  double *y = (double *)malloc(sizeof(double) * (size_t)N);
  if (!Jc || !e || !y) { free(Jc); free(e); free(y); return E_OOM; }
  for (c = 0; c < n_colors && st == OK; ++c) {
    for (j = 0; j < N; ++j) e[j] = (colors[j] == c) ? 1.0 : 0.0;
    st = fem_ref_hvp(m, z, e, y, flags);
    for (i = 0; i < N; ++i) Jc[i * n_colors + c] = y[i];
  }
  if (st == OK)
    for (i = 0; i < N; ++i)
      for (p = row_ptr[i]; p < row_ptr[i + 1]; ++p) vals[p] = Jc[i * n_colors + colors[col_idx[p]]];
  free(Jc); free(e); free(y);
  return st;
}

/* Element Hessian K_e[(a,i),(b,k)] = e1e2 part of E_e(u_e + e1 e_(a,i) + e2 e_(b,k)). */
static int elem_hessian(const fem_ref_mesh *m, int64_t e, const double *z, double Ke[12][12]) {
  int d = m->dim, nen = d + 1, a, i, b, k, a2, i2, st;
  double G[4][3], vol;
  hd ue[4][3], Ee;
  st = elem_geometry(m, e, G, &vol);
  if (st) return st;
  for (a = 0; a < nen; ++a)
    for (i = 0; i < d; ++i)
      for (b = 0; b < nen; ++b)
        for (k = 0; k < d; ++k) {
          for (a2 = 0; a2 < nen; ++a2)
            for (i2 = 0; i2 < d; ++i2)
              ue[a2][i2] = hd_const(z[(int64_t)m->conn[e * nen + a2] * d + i2]);
          ue[a][i].b = 1.0;
          ue[b][k].c = 1.0;
          st = elem_energy_hd(m, e, G, vol, ue, &Ee);
          if (st) return st;
          Ke[a * d + i][b * d + k] = Ee.d;
        }
  return OK;
}

/* ------------------------------------------------------------------ mean stress (f2)
 * Macroscopic stress of homogenization ("the volume average of the
 * microscopic stress"): sigma = sum_e vol_e P(H_e) / sum_e vol_e with P_ij = d psi / d H_ij
 * taken by forward-mode dual numbers on psi (seed E_ij), never a hand-derived stress.
 * Ascending element order, Neumaier-compensated sums.                                  */
int fem_ref_mean_stress(const fem_ref_mesh *m, const double *z, double *sigma, double *volume) {
  int d = m->dim, nen = d + 1, a, i, j, k, l, st;
  int64_t e;
  ksum acc[9], vs;
  memset(acc, 0, sizeof(acc));
  memset(&vs, 0, sizeof(vs));
  for (e = 0; e < m->n_elems; ++e) {
    double G[4][3], vol, lam, mu, H[3][3];
    st = elem_geometry(m, e, G, &vol);
    if (st) return st;
    elem_material(m, e, &lam, &mu);
    for (i = 0; i < d; ++i)
      for (j = 0; j < d; ++j) {
        H[i][j] = 0.0;
        for (a = 0; a < nen; ++a)
          H[i][j] += z[(int64_t)m->conn[e * nen + a] * d + i] * G[a][j];
      }
    for (k = 0; k < d; ++k)
      for (l = 0; l < d; ++l) {
        hd Hd[3][3], p;
        for (i = 0; i < d; ++i)
          for (j = 0; j < d; ++j) {
            Hd[i][j] = hd_const(H[i][j]);
            if (i == k && j == l) Hd[i][j].b = 1.0;
          }
        st = psi_hd(d, m->material, lam, mu, Hd, &p);
        if (st) return st;
        ks_add(&acc[k * d + l], vol * p.b);
      }
    ks_add(&vs, vol);
  }
  *volume = ks_val(&vs);
  for (k = 0; k < d * d; ++k) sigma[k] = ks_val(&acc[k]) / *volume;
  return OK;
}

/* ------------------------------------------------------------------ external loads (f3)
 * Consistent nodal loads of the linear load terms of the total potential energy (PAPER.md
 * §6.1): f_a = int N_a t dGamma over boundary facets (Line2 in 2D, Tri3 in 3D) and
 * f_a = int N_a b dOmega over the elements, by Gauss rules exact for the linear integrands
 * (Line2: 2 points xi = 1/2 -+ 1/(2 sqrt 3), w 1/2; Tri3: the 3 edge midpoints, w 1/3;
 * Tri3 element: the same; Tet4: 4 points a = (5 - sqrt 5)/20, b = (5 + 3 sqrt 5)/20, w 1/4),
 * i.e. not the one-point shortcut the GPU uses.  Accumulated in ascending facet order.     */
int fem_ref_traction_load(int dim, int64_t n_nodes, const double *coords, int64_t nf,
                          const int32_t *facets, const double *t, double *f) {
  int64_t q;
  int a, i, g;
  for (q = 0; q < nf; ++q) {
    double area, N[3][3], w[3];
    int ng;
    const int32_t *nd = facets + q * dim;
    for (a = 0; a < dim; ++a)
      if (nd[a] < 0 || nd[a] >= n_nodes) return E_ARG;
    if (dim == 2) {
      const double dx = coords[nd[1] * 2] - coords[nd[0] * 2];
      const double dy = coords[nd[1] * 2 + 1] - coords[nd[0] * 2 + 1];
      const double r = 0.5 / sqrt(3.0);
      area = sqrt(dx * dx + dy * dy);
      ng = 2;
      N[0][0] = 1.0 - (0.5 - r); N[0][1] = 0.5 - r;
      N[1][0] = 1.0 - (0.5 + r); N[1][1] = 0.5 + r;
      w[0] = w[1] = 0.5;
    } else {
      double e1[3], e2[3], c[3];
      for (i = 0; i < 3; ++i) {
        e1[i] = coords[nd[1] * 3 + i] - coords[nd[0] * 3 + i];
        e2[i] = coords[nd[2] * 3 + i] - coords[nd[0] * 3 + i];
      }
      c[0] = e1[1] * e2[2] - e1[2] * e2[1];
      c[1] = e1[2] * e2[0] - e1[0] * e2[2];
      c[2] = e1[0] * e2[1] - e1[1] * e2[0];
      area = 0.5 * sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
      ng = 3;  /* edge midpoints: N = (1/2, 1/2, 0) and permutations */
      for (g = 0; g < 3; ++g)
        for (a = 0; a < 3; ++a) N[g][a] = (a == g) ? 0.0 : 0.5;
      w[0] = w[1] = w[2] = 1.0 / 3.0;
    }
    for (g = 0; g < ng; ++g)
      for (a = 0; a < dim; ++a)
        for (i = 0; i < dim; ++i) f[(int64_t)nd[a] * dim + i] += w[g] * N[g][a] * area * t[q * dim + i];
  }
  return OK;
}

int fem_ref_body_load(const fem_ref_mesh *m, const double *b, double *f) {
  int d = m->dim, nen = d + 1, a, i, g, st;
  int64_t e;
  const double ta = (5.0 - sqrt(5.0)) / 20.0, tb = (5.0 + 3.0 * sqrt(5.0)) / 20.0;
  for (e = 0; e < m->n_elems; ++e) {
    double G[4][3], vol, N[4][4], w;
    int ng;
    st = elem_geometry(m, e, G, &vol);
    if (st) return st;
    if (d == 2) {
      ng = 3;
      w = 1.0 / 3.0;
      for (g = 0; g < 3; ++g)
        for (a = 0; a < 3; ++a) N[g][a] = (a == g) ? 0.0 : 0.5;
    } else {
      ng = 4;
      w = 0.25;
      for (g = 0; g < 4; ++g)
        for (a = 0; a < 4; ++a) N[g][a] = (a == g) ? tb : ta;
    }
    for (g = 0; g < ng; ++g)
      for (a = 0; a < nen; ++a)
        for (i = 0; i < d; ++i)
          f[(int64_t)m->conn[e * nen + a] * d + i] += w * N[g][a] * vol * b[i];
  }
  return OK;
}

/* ------------------------------------------------------------------ virtual work (f4)
 * Non-variational path (§3.1; advection-diffusion P:772-802) on a P1
 * mesh, scalar field c: W(c, v) = sum_e vol_e [ D grad c . grad v + (w_e . grad c) vbar_e ]
 * + m sum_a V_a (c_a - cold_a) v_a (reading R8: one-point rule, vbar_e = mean of
 * v over the element's nodes, w_e = mean nodal velocity, V_a = sum_{e ∋ a} vol_e/(d+1)).
 * r = grad_v W at v = 0 by dual numbers seeded on one nodal v_a at a time; the JVP
 * K x = d r(c + t x)/dt by hyper-dual numbers (eps1 on v_a, eps2 on c along x) — the
 * definitions differentiated, never a hand-assembled operator.                          */
static hd vw_elem(const fem_ref_vw *p, const fem_ref_mesh *gm, int64_t e, const hd *ce,
                  const hd *ve, int *st) {
  int d = p->dim, nen = d + 1, a, j;
  double G[4][3], vol, w[3] = {0, 0, 0};
  hd gc[3], gv[3], diff = hd_const(0.0), adv = hd_const(0.0), vbar = hd_const(0.0);
  *st = elem_geometry(gm, e, G, &vol);
  for (a = 0; a < nen; ++a)
    for (j = 0; j < d; ++j) w[j] += p->velocity[(int64_t)p->conn[e * nen + a] * d + j] / nen;
  for (j = 0; j < d; ++j) {
    gc[j] = hd_const(0.0);
    gv[j] = hd_const(0.0);
    for (a = 0; a < nen; ++a) {
      gc[j] = hd_add(gc[j], hd_scale(ce[a], G[a][j]));
      gv[j] = hd_add(gv[j], hd_scale(ve[a], G[a][j]));
    }
    diff = hd_add(diff, hd_mul(gc[j], gv[j]));
    adv = hd_add(adv, hd_scale(gc[j], w[j]));
  }
  for (a = 0; a < nen; ++a) vbar = hd_add(vbar, hd_scale(ve[a], 1.0 / nen));
  return hd_scale(hd_add(hd_scale(diff, p->diffusivity), hd_mul(adv, vbar)), vol);
}

static void vw_mesh(const fem_ref_vw *p, fem_ref_mesh *gm) {
  memset(gm, 0, sizeof(*gm));
  gm->dim = p->dim;
  gm->n_nodes = p->n_nodes;
  gm->n_elems = p->n_elems;
  gm->coords = p->coords;
  gm->conn = p->conn;
}

/* mode 0: residual of c (c_old may be NULL), mode 1: K x */
static int vw_eval(const fem_ref_vw *p, const double *c, const double *cold, double *out,
                   unsigned flags, int mode) {
  int d = p->dim, nen = d + 1, a, b, st;
  int64_t e, i;
  fem_ref_mesh gm;
  unsigned char *dir = (unsigned char *)calloc((size_t)p->n_nodes, 1);
  double *V = (double *)calloc((size_t)p->n_nodes, sizeof(double));
  if (!dir || !V) { free(dir); free(V); return E_ARG; }
  for (i = 0; i < p->n_dirichlet; ++i) dir[p->dirichlet_nodes[i]] = 1;
  const int mask = (flags & FEM_REF_APPLY_BC) && p->n_dirichlet > 0;
  vw_mesh(p, &gm);
  for (i = 0; i < p->n_nodes; ++i) out[i] = 0.0;
  for (e = 0; e < p->n_elems; ++e) {
    hd ce[4], ve[4];
    double G[4][3], vol;
    st = elem_geometry(&gm, e, G, &vol);
    if (st) { free(dir); free(V); return st; }
    for (a = 0; a < nen; ++a) V[p->conn[e * nen + a]] += vol / nen;
    for (a = 0; a < nen; ++a) {           /* seed v_a */
      for (b = 0; b < nen; ++b) {
        const int64_t n = p->conn[e * nen + b];
        double q = c[n];
        if (mode == 1 && mask && dir[n]) q = 0.0;      /* P_f x */
        ce[b] = mode == 0 ? hd_const(q) : (hd){0.0, 0.0, q, 0.0};
        ve[b] = hd_const(0.0);
        if (b == a) ve[b].b = 1.0;
      }
      hd W = vw_elem(p, &gm, e, ce, ve, &st);
      out[p->conn[e * nen + a]] += mode == 0 ? W.b : W.d;
    }
  }
  for (i = 0; i < p->n_nodes; ++i) {
    double q = c[i];
    if (mode == 1 && mask && dir[i]) q = 0.0;
    out[i] += p->mass_coef * V[i] * (q - (mode == 0 && cold ? cold[i] : 0.0));
    if (mask && dir[i]) out[i] = (mode == 0) ? 0.0 : c[i];   /* r[D] = 0; P_D x */
  }
  free(dir);
  free(V);
  return OK;
}

int fem_ref_vw_residual(const fem_ref_vw *p, const double *c, const double *cold, double *r,
                        unsigned flags) {
  return vw_eval(p, c, cold, r, flags, 0);
}

int fem_ref_vw_jvp(const fem_ref_vw *p, const double *x, double *y, unsigned flags) {
  return vw_eval(p, x, NULL, y, flags, 1);
}

static int64_t find_col(const int32_t *col_idx, int64_t lo, int64_t hi, int64_t col) {
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (col_idx[mid] < col) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* ------------------------------------------------------------------ O-elemK
 * The same sparse tangent by scatter-add of element Hessians, used as
 * an independent check of Alg. 2 and (row-sampled) at large sizes.                  */
int fem_ref_assemble_elem(const fem_ref_mesh *m, const double *z, const int64_t *row_ptr,
                          const int32_t *col_idx, double *vals, unsigned flags) {
  int d = m->dim, nen = d + 1, a, i, b, k, st;
  int64_t e, nu = n_u(m), N = n_tot(m), p, row;
  double Ke[12][12];
  unsigned char *mask = dirichlet_mask(m);
  if (!mask) return E_OOM;
  memset(vals, 0, sizeof(double) * (size_t)row_ptr[N]);
  for (e = 0; e < m->n_elems; ++e) {
    st = elem_hessian(m, e, z, Ke);
    if (st) { free(mask); return st; }
    for (a = 0; a < nen; ++a)
      for (i = 0; i < d; ++i) {
        row = (int64_t)m->conn[e * nen + a] * d + i;
        for (b = 0; b < nen; ++b)
          for (k = 0; k < d; ++k) {
            int64_t col = (int64_t)m->conn[e * nen + b] * d + k;
            p = find_col(col_idx, row_ptr[row], row_ptr[row + 1], col);
            vals[p] += Ke[a * d + i][b * d + k];
          }
      }
  }
  for (k = 0; k < m->n_mpc; ++k) {
    int64_t s = m->mpc_slave[k], ms = m->mpc_master[k], lr = nu + k;
    vals[find_col(col_idx, row_ptr[s], row_ptr[s + 1], lr)] += 1.0;
    vals[find_col(col_idx, row_ptr[ms], row_ptr[ms + 1], lr)] -= 1.0;
    vals[find_col(col_idx, row_ptr[lr], row_ptr[lr + 1], s)] += 1.0;
    vals[find_col(col_idx, row_ptr[lr], row_ptr[lr + 1], ms)] -= 1.0;
  }
  if (flags & FEM_REF_APPLY_BC)
    for (row = 0; row < N; ++row)
      for (p = row_ptr[row]; p < row_ptr[row + 1]; ++p)
        if (mask[row] || mask[col_idx[p]]) vals[p] = (row == col_idx[p]) ? 1.0 : 0.0;
  free(mask);
  return check_finite(vals, row_ptr[N]);
}

/* Row-sampled O-elemK: packed values of the requested rows (in pattern order).       */
int fem_ref_csr_rows(const fem_ref_mesh *m, const double *z, const int64_t *row_ptr,
                     const int32_t *col_idx, int64_t n_rows, const int64_t *rows,
                     double *vals_out, unsigned flags) {
  int d = m->dim, nen = d + 1, a, b, k, st = OK;
  int64_t *iptr = NULL, *iel = NULL, q, t, p, out = 0, nu = n_u(m);
  double Ke[12][12];
  unsigned char *mask = dirichlet_mask(m);
  if (!mask) return E_OOM;
  st = build_incidence(m, &iptr, &iel);
  if (st) { free(mask); return st; }
  for (q = 0; q < n_rows && st == OK; ++q) {
    int64_t row = rows[q], lo = row_ptr[row], hi = row_ptr[row + 1];
    for (p = lo; p < hi; ++p) vals_out[out + (p - lo)] = 0.0;
    if (row < nu) {
      int64_t node = row / d;
      int comp = (int)(row % d);
      for (t = iptr[node]; t < iptr[node + 1] && st == OK; ++t) {
        int64_t e = iel[t];
        st = elem_hessian(m, e, z, Ke);
        if (st) break;
        for (a = 0; a < nen; ++a) {
          if (m->conn[e * nen + a] != node) continue;
          for (b = 0; b < nen; ++b)
            for (k = 0; k < d; ++k) {
              int64_t col = (int64_t)m->conn[e * nen + b] * d + k;
              vals_out[out + find_col(col_idx, lo, hi, col) - lo] += Ke[a * d + comp][b * d + k];
            }
        }
      }
      for (k = 0; k < m->n_mpc; ++k) {
        if (m->mpc_slave[k] == row) vals_out[out + find_col(col_idx, lo, hi, nu + k) - lo] += 1.0;
        if (m->mpc_master[k] == row) vals_out[out + find_col(col_idx, lo, hi, nu + k) - lo] -= 1.0;
      }
    } else {
      k = (int)(row - nu);
      vals_out[out + find_col(col_idx, lo, hi, m->mpc_slave[k]) - lo] += 1.0;
      vals_out[out + find_col(col_idx, lo, hi, m->mpc_master[k]) - lo] -= 1.0;
    }
    if (flags & FEM_REF_APPLY_BC)
      for (p = lo; p < hi; ++p)
        if (mask[row] || mask[col_idx[p]]) vals_out[out + p - lo] = (row == col_idx[p]) ? 1.0 : 0.0;
    out += hi - lo;
  }
  free(mask); free(iptr); free(iel);
  return st;
}

/* ------------------------------------------------------------------ O-spmv
 * y = A x, ascending rows, ascending column accumulation.            */
int fem_ref_spmv(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *vals,
                 const double *x, double *y) {
  int64_t i, p;
  for (i = 0; i < n; ++i) {
    double s = 0.0;
    for (p = row_ptr[i]; p < row_ptr[i + 1]; ++p) s += vals[p] * x[col_idx[p]];
    y[i] = s;
  }
  return OK;
}

static double kdot(const double *a, const double *b, int64_t n) {
  ksum k = {0.0, 0.0};
  int64_t i;
  for (i = 0; i < n; ++i) ks_add(&k, a[i] * b[i]);
  return ks_val(&k);
}

static int apply_op(const fem_ref_mesh *m, int op, const double *z, const int64_t *row_ptr,
                    const int32_t *col_idx, const double *vals, const double *x, double *y) {
  if (op == 0) return fem_ref_hvp(m, z, x, y, FEM_REF_APPLY_BC);
  return fem_ref_spmv(n_tot(m), row_ptr, col_idx, vals, x, y);
}

/* ------------------------------------------------------------------ O-cg
 * Textbook Hestenes-Stiefel CG: r0 = b - A x0, p0 = r0,
 * alpha = r.r / p.Ap, x += alpha p, r -= alpha Ap, beta = r'.r' / r.r, p = r + beta p.
 * Stop when ||r||_2 <= max(rtol ||b||_2, atol); p.Ap <= 0 -> breakdown.
 * The operator is the masked HVP (op 0, the matrix-free path of P:168) or a CSR.     */
int fem_ref_cg(const fem_ref_mesh *m, int op, const double *z, const int64_t *row_ptr,
               const int32_t *col_idx, const double *vals, const double *b, double *x,
               double rtol, double atol, int max_iter, int *iters, double *res0, double *res) {
  int64_t N = n_tot(m), i;
  int st = OK, it = 0;
  double *r = (double *)malloc(sizeof(double) * (size_t)N);
  double *p = (double *)malloc(sizeof(double) * (size_t)N);
  double *Ap = (double *)malloc(sizeof(double) * (size_t)N);
  double rr, bn, tol;
  if (!r || !p || !Ap) { free(r); free(p); free(Ap); return E_OOM; }
  st = apply_op(m, op, z, row_ptr, col_idx, vals, x, Ap);
  if (st) goto done;
  for (i = 0; i < N; ++i) r[i] = b[i] - Ap[i];
  memcpy(p, r, sizeof(double) * (size_t)N);
  rr = kdot(r, r, N);
  bn = sqrt(kdot(b, b, N));
  tol = rtol * bn > atol ? rtol * bn : atol;
  *res0 = sqrt(rr);
  for (;;) {
    double pAp, alpha, rr_new, beta;
    if (sqrt(rr) <= tol) break;
    if (it >= max_iter) { st = E_NOTCONV; break; }
    st = apply_op(m, op, z, row_ptr, col_idx, vals, p, Ap);
    if (st) break;
    pAp = kdot(p, Ap, N);
    if (!(pAp > 0.0)) { st = E_BREAKDOWN; break; }
    alpha = rr / pAp;
    for (i = 0; i < N; ++i) x[i] += alpha * p[i];
    for (i = 0; i < N; ++i) r[i] -= alpha * Ap[i];
    rr_new = kdot(r, r, N);
    beta = rr_new / rr;
    for (i = 0; i < N; ++i) p[i] = r[i] + beta * p[i];
    rr = rr_new;
    ++it;
  }
  *res = sqrt(rr);
done:
  *iters = it;
  free(r); free(p); free(Ap);
  return st;
}

/* ------------------------------------------------------------------ O-newton
 * Full-step Newton on the condensed problem (Eq. 1): z starts at the
 * lift (z[D] = g); loop r = residual(z, BC); stop if ||r|| <= max(atol, rtol ||r0||);
 * solve K(z) delta = -r by CG on the masked operator (matrix-free Newton-Krylov,
 * P:665); z += delta.                                                               */
int fem_ref_newton(const fem_ref_mesh *m, double *z, double atol, double rtol, int max_iter,
                   double cg_rtol, int cg_max_iter, int *iters, int *cg_iters_total, double *res0,
                   double *res) {
  int64_t N = n_tot(m), i;
  int st = OK, it = 0, cgi, total = 0;
  double *r = (double *)malloc(sizeof(double) * (size_t)N);
  double *dz = (double *)malloc(sizeof(double) * (size_t)N);
  double nr, r0 = 0.0, c0, c1;
  if (!r || !dz) { free(r); free(dz); return E_OOM; }
  for (;;) {
    st = fem_ref_residual(m, z, r, FEM_REF_APPLY_BC);
    if (st) break;
    nr = sqrt(kdot(r, r, N));
    if (it == 0) r0 = nr;
    *res = nr;
    if (nr <= (atol > rtol * r0 ? atol : rtol * r0)) break;
    if (it >= max_iter) { st = E_NOTCONV; break; }
    for (i = 0; i < N; ++i) { r[i] = -r[i]; dz[i] = 0.0; }
    st = fem_ref_cg(m, 0, z, NULL, NULL, NULL, r, dz, cg_rtol, 0.0, cg_max_iter, &cgi, &c0, &c1);
    total += cgi;
    if (st) break;
    for (i = 0; i < N; ++i) z[i] += dz[i];
    ++it;
  }
  *iters = it;
  *cg_iters_total = total;
  *res0 = r0;
  free(r); free(dz);
  return st;
}
