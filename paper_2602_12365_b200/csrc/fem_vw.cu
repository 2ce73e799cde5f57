// fem_vw.cu — the non-variational (virtual-work) path (§3.1,
// P:224-236, and the advection-diffusion example P:772-802) on flat P1 meshes.
//
// A scalar field c with the virtual-work functional (one-point rule, reading R8)
//   W(c, v) = sum_e vol_e [ D grad c_e . grad v_e + (w_e . grad c_e) vbar_e ]
//           + m sum_a V_a (c_a - cold_a) v_a,
// vbar_e = mean of v over the element's nodes (= N_a at the centroid), w_e = mean nodal
// velocity, V_a = sum_{e ∋ a} vol_e / (d+1) (nodal lumped volume), m = 1/dt (0: steady).
// r(c) = grad_v W |_{v=0} and the tangent K = grad_c r (non-symmetric through the
// advection term) applied to a vector: the JVP.  Both are affine / linear in c, evaluated by
// one element kernel: y_a = sum_e vol_e [ D grad q . G_a + (w_e . grad q) / (d+1) ]
// + m V_a q_a for q = c (residual, minus m V cold) or q = x (JVP).  Dirichlet nodes by the
// masked operator (as fem_hvp: y = P_f K P_f x + P_D x; r[D] = 0).  Solved by restarted
// GMRES (CG / MINRES need symmetry): Arnoldi with classical Gram-Schmidt applied twice,
// Givens rotations on the host, x += V y at every restart.
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "element.cuh"
#include "fem_internal.cuh"

namespace fem {

struct VwProblem {
  int dim = 0;
  int64_t n_nodes = 0, n_elems = 0, n_dir = 0;
  double D = 0.0, m = 0.0;
  double *coords = nullptr, *vel = nullptr, *lumped = nullptr, *dir_vals = nullptr;
  int32_t *conn = nullptr, *dir_nodes = nullptr;
  uint8_t *is_dir = nullptr;
  double *work = nullptr;     // GMRES basis and scratch
  int64_t work_n = 0;
  double *part = nullptr;     // dot partials [kMaxDots][kReduceBlocks]
  double *dots = nullptr;     // [kMaxDots]
  int *d_err = nullptr;
};

constexpr int kVwMaxRestart = 64;

template <int D>
__global__ void k_vw_apply(const double *coords, const int32_t *conn, int64_t E,
                           const double *vel, double Dc, const double *q, const uint8_t *mask,
                           double *y) {
  constexpr int NEN = D + 1;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    int32_t nd[NEN];
    double x[NEN][D], G[NEN][D], vol, qa[NEN], w[D];
#pragma unroll
    for (int i = 0; i < D; ++i) w[i] = 0.0;
#pragma unroll
    for (int a = 0; a < NEN; ++a) {
      nd[a] = conn[e * NEN + a];
      qa[a] = (mask && mask[nd[a]]) ? 0.0 : q[nd[a]];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        x[a][i] = coords[(int64_t)nd[a] * D + i];
        w[i] += vel[(int64_t)nd[a] * D + i] * (1.0 / NEN);
      }
    }
    geometry<D>(x, G, vol);
    double gq[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double t = 0.0;
#pragma unroll
      for (int a = 0; a < NEN; ++a) t = fma(qa[a], G[a][j], t);
      gq[j] = t;
    }
    double adv = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) adv = fma(w[j], gq[j], adv);
    adv *= vol / NEN;
#pragma unroll
    for (int a = 0; a < NEN; ++a) {
      double t = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) t = fma(gq[j], G[a][j], t);
      atomicAdd(y + nd[a], fma(Dc * vol, t, adv));
    }
  }
}

// y += m V (q - qold) (qold may be null); masked rows: y = q (JVP) / 0 (residual)
__global__ void k_vw_nodal(const double *lumped, double m, const double *q, const double *qold,
                           const uint8_t *mask, int identity, int64_t n, double *y) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n;
       a += (int64_t)gridDim.x * blockDim.x) {
    if (mask && mask[a]) {
      y[a] = identity ? q[a] : 0.0;
      continue;
    }
    y[a] += m * lumped[a] * (q[a] - (qold ? qold[a] : 0.0));
  }
}

template <int D>
__global__ void k_vw_lumped(const double *coords, const int32_t *conn, int64_t E, double *V) {
  constexpr int NEN = D + 1;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    double x[NEN][D], G[NEN][D], vol;
#pragma unroll
    for (int a = 0; a < NEN; ++a)
#pragma unroll
      for (int i = 0; i < D; ++i) x[a][i] = coords[(int64_t)conn[e * NEN + a] * D + i];
    geometry<D>(x, G, vol);
#pragma unroll
    for (int a = 0; a < NEN; ++a) atomicAdd(V + conn[e * NEN + a], vol / NEN);
  }
}

__global__ void k_vw_check(const int32_t *conn, int64_t E, int64_t n, int dim, int *err) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int nen = dim + 1;
    for (int a = 0; a < nen; ++a) {
      const int32_t v = conn[e * nen + a];
      if (v < 0 || v >= n) atomicOr(err, 16);
    }
  }
}

static fem_status vw_apply(VwProblem *p, const double *q, const double *qold, double *y,
                           bool bc, bool identity, cudaStream_t s) {
  FEM_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * p->n_nodes, s));
  const uint8_t *mask = bc ? p->is_dir : nullptr;
  if (p->n_elems) {
    const int g = grid_for(p->n_elems);
    if (p->dim == 2) k_vw_apply<2><<<g, kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->vel, p->D, q, mask, y);
    else k_vw_apply<3><<<g, kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->vel, p->D, q, mask, y);
  }
  k_vw_nodal<<<grid_for(p->n_nodes), kThreads, 0, s>>>(p->lumped, p->m, q, qold, mask,
                                                      identity ? 1 : 0, p->n_nodes, y);
  FEM_LAUNCH_CHECK("virtual-work apply");
  return FEM_OK;
}

// ------------------------------------------------------------------ GMRES helpers
// dots[i] = sum_k V_i[k] w[k] for i < j (partials per block, fixed-order final sum)
__global__ void k_multi_dot(const double *V, int64_t n, int j, const double *w, double *part) {
  for (int i = 0; i < j; ++i) {
    double acc = 0.0;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
      acc = fma(V[(int64_t)i * n + k], w[k], acc);
    const double t = block_sum<kThreads>(acc);
    if (threadIdx.x == 0) part[(int64_t)i * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void k_multi_final(const double *part, int nb, int j, double *dots) {
  for (int i = 0; i < j; ++i) {
    double a = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) a += part[(int64_t)i * nb + b];
    const double t = block_sum<kThreads>(a);
    if (threadIdx.x == 0) dots[i] = t;
  }
}

// w -= sum_i h_i V_i
__global__ void k_multi_axpy(const double *V, int64_t n, int j, const double *h, double *w) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    double t = w[k];
    for (int i = 0; i < j; ++i) t = fma(-h[i], V[(int64_t)i * n + k], t);
    w[k] = t;
  }
}

__global__ void k_vw_sub(const double *a, const double *b, double *out, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    out[k] = a[k] - b[k];
}

__global__ void k_scale_into(const double *a, double s, double *b, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    b[k] = s * a[k];
}

}  // namespace fem

using namespace fem;

struct fem_vw_problem {
  fem::VwProblem p;
};

static fem_status vw_dots(VwProblem *p, const double *V, int j, const double *w, double *host,
                          cudaStream_t s) {
  const int nb = grid_for(p->n_nodes, kThreads, 296);
  k_multi_dot<<<nb, kThreads, 0, s>>>(V, p->n_nodes, j, w, p->part);
  k_multi_final<<<1, kThreads, 0, s>>>(p->part, nb, j, p->dots);
  FEM_LAUNCH_CHECK("gmres dots");
  FEM_CUDA(cudaMemcpyAsync(host, p->dots, sizeof(double) * j, cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  return FEM_OK;
}

extern "C" {

fem_status fem_vw_create(fem_vw_problem **out, const fem_vw_desc *d, fem_stream stream) {
  FEM_NVTX_RANGE("fem_vw_create");
  FEM_ARG(out && d, "fem_vw_create: null argument");
  FEM_ARG(d->dim == 2 || d->dim == 3, "fem_vw_create: dim must be 2 or 3");
  FEM_ARG(d->n_nodes > 0 && d->n_elems >= 0 && d->coords && (d->n_elems == 0 || d->conn) && d->velocity,
          "fem_vw_create: mesh arrays");
  FEM_ARG(d->diffusivity >= 0.0 && d->mass_coef >= 0.0, "fem_vw_create: D, m >= 0");
  FEM_ARG(d->n_dirichlet >= 0 && (d->n_dirichlet == 0 || (d->dirichlet_nodes && d->dirichlet_vals)),
          "fem_vw_create: Dirichlet arrays");
  cudaStream_t s = (cudaStream_t)stream;
  auto *h = new fem_vw_problem();
  VwProblem *p = &h->p;
  p->dim = d->dim; p->n_nodes = d->n_nodes; p->n_elems = d->n_elems; p->n_dir = d->n_dirichlet;
  p->D = d->diffusivity; p->m = d->mass_coef;
  const int D = d->dim;
  auto fail = [&](fem_status st) { fem_vw_destroy(h); return st; };
#define VW_C(call) do { cudaError_t e_ = (call); if (e_ != cudaSuccess) return fail(cuda_status(e_, #call)); } while (0)
  VW_C(cudaMalloc(&p->coords, sizeof(double) * D * p->n_nodes));
  VW_C(cudaMalloc(&p->vel, sizeof(double) * D * p->n_nodes));
  VW_C(cudaMalloc(&p->lumped, sizeof(double) * p->n_nodes));
  VW_C(cudaMalloc(&p->conn, sizeof(int32_t) * (D + 1) * (p->n_elems > 0 ? p->n_elems : 1)));
  VW_C(cudaMalloc(&p->is_dir, p->n_nodes));
  VW_C(cudaMalloc(&p->d_err, sizeof(int)));
  VW_C(cudaMalloc(&p->part, sizeof(double) * (kVwMaxRestart + 1) * 296));
  VW_C(cudaMalloc(&p->dots, sizeof(double) * (kVwMaxRestart + 1)));
  VW_C(cudaMemcpyAsync(p->coords, d->coords, sizeof(double) * D * p->n_nodes, cudaMemcpyDefault, s));
  VW_C(cudaMemcpyAsync(p->vel, d->velocity, sizeof(double) * D * p->n_nodes, cudaMemcpyDefault, s));
  if (p->n_elems)
    VW_C(cudaMemcpyAsync(p->conn, d->conn, sizeof(int32_t) * (D + 1) * p->n_elems, cudaMemcpyDefault, s));
  VW_C(cudaMemsetAsync(p->is_dir, 0, p->n_nodes, s));
  VW_C(cudaMemsetAsync(p->lumped, 0, sizeof(double) * p->n_nodes, s));
  VW_C(cudaMemsetAsync(p->d_err, 0, sizeof(int), s));
  if (p->n_dir) {
    VW_C(cudaMalloc(&p->dir_nodes, sizeof(int32_t) * p->n_dir));
    VW_C(cudaMalloc(&p->dir_vals, sizeof(double) * p->n_dir));
    VW_C(cudaMemcpyAsync(p->dir_nodes, d->dirichlet_nodes, sizeof(int32_t) * p->n_dir, cudaMemcpyDefault, s));
    VW_C(cudaMemcpyAsync(p->dir_vals, d->dirichlet_vals, sizeof(double) * p->n_dir, cudaMemcpyDefault, s));
    std::vector<int32_t> hn(p->n_dir);
    VW_C(cudaMemcpyAsync(hn.data(), d->dirichlet_nodes, sizeof(int32_t) * p->n_dir, cudaMemcpyDefault, s));
    VW_C(cudaStreamSynchronize(s));
    std::vector<uint8_t> mask(p->n_nodes, 0);
    for (int32_t v : hn) {
      if (v < 0 || v >= p->n_nodes) { set_error("fem_vw_create: Dirichlet node out of range"); return fail(FEM_ERR_INVALID_ARG); }
      mask[v] = 1;
    }
    VW_C(cudaMemcpyAsync(p->is_dir, mask.data(), p->n_nodes, cudaMemcpyHostToDevice, s));
  }
  int herr = 0;
  if (p->n_elems) {
    k_vw_check<<<grid_for(p->n_elems), kThreads, 0, s>>>(p->conn, p->n_elems, p->n_nodes, D, p->d_err);
    VW_C(cudaMemcpyAsync(&herr, p->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
    VW_C(cudaStreamSynchronize(s));
    if (herr) { set_error("fem_vw_create: element node id out of range"); return fail(FEM_ERR_INVALID_ARG); }
    if (D == 2) k_vw_lumped<2><<<grid_for(p->n_elems), kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lumped);
    else k_vw_lumped<3><<<grid_for(p->n_elems), kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lumped);
  }
  VW_C(cudaStreamSynchronize(s));
#undef VW_C
  *out = h;
  return FEM_OK;
}

fem_status fem_vw_destroy(fem_vw_problem *h) {
  FEM_NVTX_RANGE("fem_vw_destroy");
  if (!h) return FEM_OK;
  VwProblem *p = &h->p;
  void *b[] = {p->coords, p->vel, p->lumped, p->dir_vals, p->conn, p->dir_nodes, p->is_dir,
               p->work, p->part, p->dots, p->d_err};
  for (void *x : b)
    if (x) cudaFree(x);
  delete h;
  return FEM_OK;
}

__global__ void k_vw_lift(const int32_t *nodes, const double *vals, int64_t n, double *c) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    c[nodes[q]] = vals[q];
}

fem_status fem_vw_apply_dirichlet(fem_vw_problem *h, double *c, fem_stream stream) {
  FEM_NVTX_RANGE("fem_vw_apply_dirichlet");
  FEM_ARG(h && c, "fem_vw_apply_dirichlet: null argument");
  VwProblem *p = &h->p;
  if (p->n_dir)
    k_vw_lift<<<grid_for(p->n_dir), kThreads, 0, (cudaStream_t)stream>>>(p->dir_nodes, p->dir_vals, p->n_dir, c);
  FEM_LAUNCH_CHECK("vw lift");
  return FEM_OK;
}

fem_status fem_vw_residual(fem_vw_problem *h, const double *c, const double *c_old, double *r,
                           unsigned flags, fem_stream stream) {
  FEM_NVTX_RANGE("fem_vw_residual");
  FEM_ARG(h && c && r, "fem_vw_residual: null argument");
  FEM_ARG(c != r, "fem_vw_residual: c and r alias");
  VwProblem *p = &h->p;
  // r = K c - m V c_old; the residual must see the lifted c, so no input masking here
  cudaStream_t s = (cudaStream_t)stream;
  fem_status st = vw_apply(p, c, c_old, r, false, false, s);
  if (st) return st;
  if ((flags & FEM_APPLY_BC) && p->n_dir) {
    // r[D] = 0: the nodal kernel with m = 0 and identity = 0 zeroes the constrained rows
    k_vw_nodal<<<grid_for(p->n_nodes), kThreads, 0, s>>>(p->lumped, 0.0, r, nullptr, p->is_dir, 0, p->n_nodes, r);
    FEM_LAUNCH_CHECK("vw residual bc");
  }
  return FEM_OK;
}

fem_status fem_vw_jvp(fem_vw_problem *h, const double *x, double *y, unsigned flags,
                      fem_stream stream) {
  FEM_NVTX_RANGE("fem_vw_jvp");
  FEM_ARG(h && x && y, "fem_vw_jvp: null argument");
  FEM_ARG(x != y, "fem_vw_jvp: x and y alias");
  VwProblem *p = &h->p;
  const bool bc = (flags & FEM_APPLY_BC) && p->n_dir;
  return vw_apply(p, x, nullptr, y, bc, bc, (cudaStream_t)stream);
}

fem_status fem_vw_gmres_solve(fem_vw_problem *h, const double *b, double *x,
                              const fem_gmres_opts *o, fem_cg_report *rep, fem_stream stream) {
  FEM_NVTX_RANGE("fem_vw_gmres_solve");
  FEM_ARG(h && b && x && o && rep, "fem_vw_gmres_solve: null argument");
  FEM_ARG(o->restart >= 1 && o->restart <= kVwMaxRestart, "fem_vw_gmres_solve: restart in [1, 64]");
  VwProblem *p = &h->p;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = p->n_nodes;
  const int mr = o->restart;
  const bool bc = p->n_dir > 0;
  if (p->work_n < (int64_t)(mr + 2) * n) {
    if (p->work) cudaFree(p->work);
    p->work = nullptr;
    FEM_CUDA(cudaMalloc(&p->work, sizeof(double) * (size_t)(mr + 2) * n));
    p->work_n = (int64_t)(mr + 2) * n;
  }
  double *V = p->work, *w = p->work + (int64_t)(mr + 1) * n;
  const int g = grid_for(n);
  double hb = 0.0;
  fem_status st = vw_dots(p, b, 1, b, &hb, s);
  if (st) return st;
  const double tol = std::fmax(o->rtol * std::sqrt(hb), o->atol);
  std::vector<double> H((size_t)(mr + 1) * mr), cs(mr), sn(mr), gv(mr + 1), hc(mr + 1);
  rep->iters = 0;
  rep->converged = 0;
  double beta = 0.0;
  fem_status result = FEM_OK;
  for (int cycle = 0;; ++cycle) {
    // r = b - A x into V_0
    st = vw_apply(p, x, nullptr, w, bc, bc, s);
    if (st) return st;
    k_vw_sub<<<g, kThreads, 0, s>>>(b, w, V, n);
    FEM_LAUNCH_CHECK("gmres restart");
    st = vw_dots(p, V, 1, V, &beta, s);
    if (st) return st;
    beta = std::sqrt(beta);
    if (cycle == 0) rep->res0 = beta;
    rep->res = beta;
    if (beta <= tol) { rep->converged = 1; break; }
    if (rep->iters >= o->max_iter) { result = FEM_ERR_NOT_CONVERGED; break; }
    k_scale_into<<<g, kThreads, 0, s>>>(V, 1.0 / beta, V, n);
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int j = 0;
    for (; j < mr && rep->iters < o->max_iter; ++j) {
      double *vj1 = V + (int64_t)(j + 1) * n;
      st = vw_apply(p, V + (int64_t)j * n, nullptr, vj1, bc, bc, s);
      if (st) return st;
      // classical Gram-Schmidt, twice
      for (int i = 0; i <= j; ++i) H[(size_t)i * mr + j] = 0.0;
      for (int pass = 0; pass < 2; ++pass) {
        st = vw_dots(p, V, j + 1, vj1, hc.data(), s);
        if (st) return st;
        FEM_CUDA(cudaMemcpyAsync(p->dots, hc.data(), sizeof(double) * (j + 1), cudaMemcpyHostToDevice, s));
        k_multi_axpy<<<g, kThreads, 0, s>>>(V, n, j + 1, p->dots, vj1);
        FEM_LAUNCH_CHECK("gmres orthogonalize");
        for (int i = 0; i <= j; ++i) H[(size_t)i * mr + j] += hc[i];
      }
      double hn = 0.0;
      st = vw_dots(p, vj1, 1, vj1, &hn, s);
      if (st) return st;
      hn = std::sqrt(hn);
      H[(size_t)(j + 1) * mr + j] = hn;
      if (hn > 0.0) k_scale_into<<<g, kThreads, 0, s>>>(vj1, 1.0 / hn, vj1, n);
      // apply the previous rotations, then a new one
      for (int i = 0; i < j; ++i) {
        const double a = H[(size_t)i * mr + j], c2 = H[(size_t)(i + 1) * mr + j];
        H[(size_t)i * mr + j] = cs[i] * a + sn[i] * c2;
        H[(size_t)(i + 1) * mr + j] = -sn[i] * a + cs[i] * c2;
      }
      const double a = H[(size_t)j * mr + j], c2 = H[(size_t)(j + 1) * mr + j];
      const double rr = std::hypot(a, c2);
      cs[j] = rr > 0.0 ? a / rr : 1.0;
      sn[j] = rr > 0.0 ? c2 / rr : 0.0;
      H[(size_t)j * mr + j] = rr;
      H[(size_t)(j + 1) * mr + j] = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      ++rep->iters;
      rep->res = std::fabs(gv[j + 1]);
      if (rep->res <= tol || hn == 0.0) { ++j; break; }
    }
    // y = R^{-1} g ; x += V y
    std::vector<double> y(j, 0.0);
    for (int i = j - 1; i >= 0; --i) {
      double t = gv[i];
      for (int k = i + 1; k < j; ++k) t -= H[(size_t)i * mr + k] * y[k];
      y[i] = t / H[(size_t)i * mr + i];
    }
    for (int i = 0; i < j; ++i) y[i] = -y[i];  // k_multi_axpy subtracts
    FEM_CUDA(cudaMemcpyAsync(p->dots, y.data(), sizeof(double) * j, cudaMemcpyHostToDevice, s));
    k_multi_axpy<<<g, kThreads, 0, s>>>(V, n, j, p->dots, x);
    FEM_LAUNCH_CHECK("gmres update");
    FEM_CUDA(cudaStreamSynchronize(s));
  }
  if (result == FEM_ERR_NOT_CONVERGED) set_error("GMRES: iteration cap reached");
  return result;
}

}  // extern "C"
