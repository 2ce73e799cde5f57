// element.cuh — per-element math of the hot path (device functions, templated on dim).
//
// One-point P1 simplex (Eq. 2; reading C4): H = sum_a u_a (x) G_a is
// constant per element, Psi_e = vol * psi(H).  Hand-derived derivatives (north_star:
// "derivatives are hand-derived per energy density rather than produced by an AD
// framework"):
//   residual  f_a = vol * P(H) G_a,             P = d psi / dH           (Eq. 1)
//   HVP       y_a = vol * dP(H)[dH] G_a,        dH = sum_a v_a (x) G_a   (Eq. 3)
// Linear elastic (plane strain in 2D, reading C2):
//   psi = mu eps:eps + lambda/2 tr(eps)^2, P = mu (H + H^T) + lambda tr(H) I,
//   dP = mu (dH + dH^T) + lambda tr(dH) I.
// Compressible neo-Hookean (reading C1):
//   psi = mu/2 (F:F - d - 2 ln J) + lambda/2 (ln J)^2, F = I + H, J = det F,
//   P  = mu F + (lambda ln J - mu) F^{-T},
//   dP = mu dH + (mu - lambda ln J) F^{-T} dH^T F^{-T} + lambda (F^{-T}:dH) F^{-T}.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fem {

#ifndef FEM_FAST_MATH
#define FEM_FAST_MATH 1
#endif

// 1/x to ~1 ulp: the SFU's ~2^-23 seed (rcp.approx.ftz.f64) refined by two Newton steps
// (quadratic convergence: 2^-46, then below 2^-53 + one rounding).  For the finite,
// nonzero geometric determinants of the element kernels (DegenerateElement rejects
// det <= eps_det at create; inverted deformed elements are flagged before use); the
// compiler's IEEE 1.0/x adds a slow-path branch for denormal / special operands.
__device__ __forceinline__ double fem_rcp(double x) {
#if FEM_FAST_MATH
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#else
  return 1.0 / x;
#endif
}

// ln x for x > 0: x = 2^k m with m in [sqrt(1/2), sqrt(2)), ln m = 2 atanh(f),
// f = (m - 1)/(m + 1), |f| <= 0.1716, atanh(f)/f = sum_{j<=11} f^2j / (2j + 1) (truncation
// below 2^-55 relative); ln x = k ln 2 + ln m with ln 2 split hi/lo.  ~30 instructions
// against ~65 for the general log(); zero, negative, subnormal, inf and NaN operands take
// log() itself (same results as libm there).
// FEM_LOG_CTAB: the series coefficients and ln 2 hi/lo come from a __constant__ table (read
// as uniform-register pairs, LDCU.128) instead of two UMOV immediates per coefficient at every
// use (SASS of the NH HVP: 48 UMOV among ~550 phase-1 instructions), and the series stops at
// 1/21: |f| <= 0.1716, so the first dropped term of ln m = 2f (1 + s P(s)) is s^11 / 23 <
// 1e-18 relative.  Measured neutral (r02, cfg 3: HVP 0.916 vs 0.908 ms, energy 0.377 vs 0.381):
// the table's LDCU loads sit on the log's critical path where the immediates did not; off.
#ifndef FEM_LOG_CTAB
#define FEM_LOG_CTAB 0
#endif
#if FEM_LOG_CTAB
static __constant__ double kFemLogC[12] = {
    1.0 / 21.0, 1.0 / 19.0, 1.0 / 17.0, 1.0 / 15.0, 1.0 / 13.0, 1.0 / 11.0,
    1.0 / 9.0,  1.0 / 7.0,  1.0 / 5.0,  1.0 / 3.0,  6.93147180369123816490e-01,
    1.90821492927058770002e-10};
#endif
__device__ __forceinline__ double fem_log(double x) {
#if FEM_FAST_MATH
  const int hi = __double2hiint(x);
  if (hi < 0x00100000 || hi >= 0x7ff00000) return log(x);
  int k = (hi >> 20) - 1023;
  int mh = (hi & 0x000fffff) | 0x3ff00000;
  if (mh > 0x3ff6a09e) {  // m > sqrt(2): halve it
    mh -= 0x00100000;
    ++k;
  }
  const double m = __hiloint2double(mh, __double2loint(x));
  const double f = (m - 1.0) * fem_rcp(m + 1.0);
  const double s = f * f;
#if FEM_LOG_CTAB
  double p = kFemLogC[0];
#pragma unroll
  for (int j = 1; j < 10; ++j) p = fma(p, s, kFemLogC[j]);
  const double lnm = fma(2.0 * f * s, p, 2.0 * f);   // 2f + 2f s P(s)
  const double dk = (double)k;
  return fma(dk, kFemLogC[10], fma(dk, kFemLogC[11], lnm));
#else
  double p = 1.0 / 23.0;
  p = fma(p, s, 1.0 / 21.0);
  p = fma(p, s, 1.0 / 19.0);
  p = fma(p, s, 1.0 / 17.0);
  p = fma(p, s, 1.0 / 15.0);
  p = fma(p, s, 1.0 / 13.0);
  p = fma(p, s, 1.0 / 11.0);
  p = fma(p, s, 1.0 / 9.0);
  p = fma(p, s, 1.0 / 7.0);
  p = fma(p, s, 1.0 / 5.0);
  p = fma(p, s, 1.0 / 3.0);
  const double lnm = fma(2.0 * f * s, p, 2.0 * f);   // 2f + 2f s P(s)
  const double dk = (double)k;
  return fma(dk, 6.93147180369123816490e-01, fma(dk, 1.90821492927058770002e-10, lnm));
#endif
#else
  return log(x);
#endif
}

template <int D>
struct Elem {
  static constexpr int NEN = D + 1;
};

// Geometry from nodal coordinates.  J = [x1-x0 | ... | xd-x0]; G_a (a>=1) = row a-1 of
// J^{-1}; G_0 = -sum G_a; vol = det J / d!.  Returns det J.
template <int D>
__device__ __forceinline__ double geometry(const double (&x)[D + 1][D], double (&G)[D + 1][D],
                                           double &vol) {
  if constexpr (D == 2) {
    const double j00 = x[1][0] - x[0][0], j01 = x[2][0] - x[0][0];
    const double j10 = x[1][1] - x[0][1], j11 = x[2][1] - x[0][1];
    const double det = j00 * j11 - j01 * j10;
    const double id = 1.0 / det;
    G[1][0] = j11 * id;
    G[1][1] = -j01 * id;
    G[2][0] = -j10 * id;
    G[2][1] = j00 * id;
    G[0][0] = -G[1][0] - G[2][0];
    G[0][1] = -G[1][1] - G[2][1];
    vol = 0.5 * det;
    return det;
  } else {
    double J[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) J[i][j] = x[j + 1][i] - x[0][i];
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    const double c10 = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    const double c11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    const double c12 = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    const double c20 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    const double c21 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    const double c22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    const double id = 1.0 / det;
    // inv[i][j] = cof[j][i] / det; G_{a}[j] = inv[a-1][j]
    G[1][0] = c00 * id; G[1][1] = c10 * id; G[1][2] = c20 * id;
    G[2][0] = c01 * id; G[2][1] = c11 * id; G[2][2] = c21 * id;
    G[3][0] = c02 * id; G[3][1] = c12 * id; G[3][2] = c22 * id;
#pragma unroll
    for (int j = 0; j < 3; ++j) G[0][j] = -(G[1][j] + G[2][j] + G[3][j]);
    vol = det * (1.0 / 6.0);
    return det;
  }
}

template <int D>
__device__ __forceinline__ void field_gradient(const double (&u)[D + 1][D],
                                               const double (&G)[D + 1][D], double (&H)[D][D]) {
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double h = 0.0;
#pragma unroll
      for (int a = 0; a < D + 1; ++a) h = fma(u[a][i], G[a][j], h);
      H[i][j] = h;
    }
}

// Scatter-ready nodal vectors out_a = vol * A G_a.
template <int D>
__device__ __forceinline__ void nodal_from_stress(const double (&A)[D][D],
                                                  const double (&G)[D + 1][D], double vol,
                                                  double (&out)[D + 1][D]) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double s0 = 0.0;
#pragma unroll
    for (int a = 1; a < D + 1; ++a) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) t = fma(A[i][j], G[a][j], t);
      out[a][i] = vol * t;
      s0 += out[a][i];
    }
    out[0][i] = -s0;
  }
}

// ---- cofactor form (tile kernels): G_a = c_a / det for a >= 1, so with vol = det / d!
// the nodal vectors are vol P G_a = (P / d!) c_a and dH = dHh / det; the scalings fold into
// the material coefficients (P and dP are linear in (lambda, mu)), and G, G_0, vol are
// never formed.
template <int D>
__device__ __forceinline__ double cof_gradients(const double (&x)[D + 1][D], double (&c)[D][D]) {
  if constexpr (D == 2) {
    const double j00 = x[1][0] - x[0][0], j01 = x[2][0] - x[0][0];
    const double j10 = x[1][1] - x[0][1], j11 = x[2][1] - x[0][1];
    c[0][0] = j11;  c[0][1] = -j01;
    c[1][0] = -j10; c[1][1] = j00;
    return j00 * j11 - j01 * j10;
  } else {
    double J[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) J[i][j] = x[j + 1][i] - x[0][i];
    // c[a-1][j] = cof(J)[j][a-1]
    c[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    c[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    c[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    c[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    c[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    c[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    c[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    c[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    c[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    return J[0][0] * c[0][0] + J[0][1] * c[1][0] + J[0][2] * c[2][0];
  }
}

// Gradients G_a from the cofactor rows with the SFU-seeded reciprocal: G_a = c_a / det
// (a >= 1), G_0 = -sum_a G_a; returns det J and 1/det J in id.
template <int D>
__device__ __forceinline__ double cof_geometry(const double (&x)[D + 1][D], double (&G)[D + 1][D],
                                               double &id) {
  double c[D][D];
  const double det = cof_gradients<D>(x, c);
  id = fem_rcp(det);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      G[a + 1][j] = c[a][j] * id;
      s += G[a + 1][j];
    }
    G[0][j] = -s;
  }
  return det;
}

// Edge form of the deformed element x + u: node 0 at the origin, node a at
// (x_a - x_0) + (u_a - u_0).  Differences first: forming x + u would round at the scale of
// |x| instead of the element size (cofactors of a 1e-3 element off by 1e-13 relative).
template <int D>
__device__ __forceinline__ void deformed_edges(const double (&x)[D + 1][D],
                                               const double (&u)[D + 1][D],
                                               double (&xd)[D + 1][D]) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    xd[0][i] = 0.0;
#pragma unroll
    for (int a = 1; a < D + 1; ++a) xd[a][i] = (x[a][i] - x[0][i]) + (u[a][i] - u[0][i]);
  }
}

// Hh = sum_{a>=1} (u_a - u_0) (x) c_a   (= det * H)
template <int D>
__device__ __forceinline__ void grad_hat(const double (&u)[D + 1][D], const double (&c)[D][D],
                                         double (&Hh)[D][D]) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double du[D];
#pragma unroll
    for (int a = 0; a < D; ++a) du[a] = u[a + 1][i] - u[0][i];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double h = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) h = fma(du[a], c[a][j], h);
      Hh[i][j] = h;
    }
  }
}

// f_a = S c_a (a >= 1), f_0 = -sum_a f_a
template <int D>
__device__ __forceinline__ void nodal_from_c(const double (&S)[D][D], const double (&c)[D][D],
                                             double (&f)[D + 1][D]) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double s0 = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) t = fma(S[i][j], c[a][j], t);
      f[a + 1][i] = t;
      s0 += t;
    }
    f[0][i] = -s0;
  }
}

// ------------------------------------------------------------------ linear elastic
template <int D>
__device__ __forceinline__ double le_psi(const double (&H)[D][D], double lam, double mu) {
  double tr = 0.0, ee = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    tr += H[i][i];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const double e = 0.5 * (H[i][j] + H[j][i]);
      ee = fma(e, e, ee);
    }
  }
  return mu * ee + 0.5 * lam * tr * tr;
}

template <int D>
__device__ __forceinline__ void le_stress(const double (&H)[D][D], double lam, double mu,
                                          double (&P)[D][D]) {
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) tr += H[i][i];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) P[i][j] = mu * (H[i][j] + H[j][i]) + (i == j ? lam * tr : 0.0);
}

// ------------------------------------------------------------------ neo-Hookean
template <int D>
struct NHState {
  double F[D][D];
  double FiT[D][D];  // F^{-T}
  double lnJ, J;
};

// Returns false when J <= 0 (inverted element).
template <int D>
__device__ __forceinline__ bool nh_state(const double (&H)[D][D], NHState<D> &s) {
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) s.F[i][j] = H[i][j] + (i == j ? 1.0 : 0.0);
  double cof[D][D];
  if constexpr (D == 2) {
    cof[0][0] = s.F[1][1];
    cof[0][1] = -s.F[1][0];
    cof[1][0] = -s.F[0][1];
    cof[1][1] = s.F[0][0];
    s.J = s.F[0][0] * s.F[1][1] - s.F[0][1] * s.F[1][0];
  } else {
    const double(&F)[3][3] = s.F;
    cof[0][0] = F[1][1] * F[2][2] - F[1][2] * F[2][1];
    cof[0][1] = F[1][2] * F[2][0] - F[1][0] * F[2][2];
    cof[0][2] = F[1][0] * F[2][1] - F[1][1] * F[2][0];
    cof[1][0] = F[0][2] * F[2][1] - F[0][1] * F[2][2];
    cof[1][1] = F[0][0] * F[2][2] - F[0][2] * F[2][0];
    cof[1][2] = F[0][1] * F[2][0] - F[0][0] * F[2][1];
    cof[2][0] = F[0][1] * F[1][2] - F[0][2] * F[1][1];
    cof[2][1] = F[0][2] * F[1][0] - F[0][0] * F[1][2];
    cof[2][2] = F[0][0] * F[1][1] - F[0][1] * F[1][0];
    s.J = F[0][0] * cof[0][0] + F[0][1] * cof[0][1] + F[0][2] * cof[0][2];
  }
  if (!(s.J > 0.0)) return false;
  const double iJ = fem_rcp(s.J);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) s.FiT[i][j] = cof[i][j] * iJ;
  s.lnJ = fem_log(s.J);
  return true;
}

template <int D>
__device__ __forceinline__ double nh_psi(const double (&H)[D][D], const NHState<D> &s,
                                         double lam, double mu) {
  // F:F - d = 2 tr H + H:H (no cancellation against d)
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    t += 2.0 * H[i][i];
#pragma unroll
    for (int j = 0; j < D; ++j) t = fma(H[i][j], H[i][j], t);
  }
  return 0.5 * mu * (t - 2.0 * s.lnJ) + 0.5 * lam * s.lnJ * s.lnJ;
}

template <int D>
__device__ __forceinline__ void nh_stress(const NHState<D> &s, double lam, double mu,
                                          double (&P)[D][D]) {
  const double c = lam * s.lnJ - mu;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) P[i][j] = fma(c, s.FiT[i][j], mu * s.F[i][j]);
}

template <int D>
__device__ __forceinline__ void nh_dstress(const NHState<D> &s, double lam, double mu,
                                           const double (&dH)[D][D], double (&dP)[D][D]) {
  // T = dH^T F^{-T};  M = F^{-T} T = F^{-T} dH^T F^{-T};  tr = F^{-T} : dH
  double T[D][D];
#pragma unroll
  for (int k = 0; k < D; ++k)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double t = 0.0;
#pragma unroll
      for (int l = 0; l < D; ++l) t = fma(dH[l][k], s.FiT[l][j], t);
      T[k][j] = t;
    }
  double tr = 0.0;  // F^{-T} : dH = tr(dH^T F^{-T}) = tr T
#pragma unroll
  for (int k = 0; k < D; ++k) tr += T[k][k];
  const double c1 = mu - lam * s.lnJ, c2 = lam * tr;
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double m = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) m = fma(s.FiT[i][k], T[k][j], m);
      dP[i][j] = fma(c2, s.FiT[i][j], fma(c1, m, mu * dH[i][j]));
    }
}

}  // namespace fem
