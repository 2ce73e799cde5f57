// fem_solve.cu — CG (a12) and Newton (a13) driven natively on the device.
//
// CG: textbook Hestenes-Stiefel with optional Jacobi.  Scalars (r.r, p.Ap,
// r.z) stay on the device in ping-pong slots so no kernel reads a value another kernel of
// the same iteration writes; the host reads ||r|| every `check_every` iterations.
// Operator: the masked HVP at z (matrix-free Newton-Krylov) or the CSR SpMV.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "fem_internal.cuh"

namespace fem {

fem_status run_assemble(Problem *p, const double *z, double *vals, unsigned flags, cudaStream_t s);

// CG scalars: for slot parity c, rz at 2c and rr at 2c + 1 (adjacent: one 2-double
// all-reduce per iteration on multi-GPU problems)
enum { S_RZ0 = 0, S_RR0 = 1, S_RZ1 = 2, S_RR1 = 3, S_PAP = 4, S_BB = 5, S_NRM = 6 };

__global__ void k_sub(const double *b, const double *Ax, double *r, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    r[i] = b[i] - Ax[i];
}

// z = dinv * r (or r), p = z, partial r.r and r.z
__global__ void k_cg_start(const double *r, const double *dinv, double *zv, double *p, int64_t n,
                           double *part_rr, double *part_rz, const uint8_t *owned, int dim) {
  double rr = 0.0, rz = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = r[i];
    const double zi = dinv ? dinv[i] * ri : ri;
    if (dinv) zv[i] = zi;
    p[i] = zi;
    if (!owned || owned[i / dim]) {
      rr = fma(ri, ri, rr);
      rz = fma(ri, zi, rz);
    }
  }
  const double a = block_sum<kThreads>(rr);
  const double b = block_sum<kThreads>(rz);
  if (threadIdx.x == 0) {
    part_rr[blockIdx.x] = a;
    part_rz[blockIdx.x] = b;
  }
}

// alpha = rz / pAp; x += alpha p; r -= alpha Ap; z = dinv r; partial r.r, r.z
__global__ void k_cg_update(const double *scal, int rz_slot, double *x, double *r, double *zv,
                            const double *p, const double *Ap, const double *dinv, int64_t n,
                            double *part_rr, double *part_rz, const uint8_t *owned, int dim) {
  const double alpha = scal[rz_slot] / scal[S_PAP];
  double rr = 0.0, rz = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, Ap[i], r[i]);
    r[i] = ri;
    const double zi = dinv ? dinv[i] * ri : ri;
    if (dinv) zv[i] = zi;
    if (!owned || owned[i / dim]) {
      rr = fma(ri, ri, rr);
      rz = fma(ri, zi, rz);
    }
  }
  const double a = block_sum<kThreads>(rr);
  const double b = block_sum<kThreads>(rz);
  if (threadIdx.x == 0) {
    part_rr[blockIdx.x] = a;
    part_rz[blockIdx.x] = b;
  }
}

// p = z + beta p, beta = rz_new / rz_old
__global__ void k_cg_dir(const double *scal, int rz_old, int rz_new, const double *zv, double *p,
                         int64_t n) {
  const double beta = scal[rz_new] / scal[rz_old];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = fma(beta, p[i], zv[i]);
}

__global__ void k_final_sum2(const double *pa, const double *pb, int n, double *oa, double *ob) {
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    a += pa[i];
    b += pb[i];
  }
  const double ta = block_sum<kThreads>(a);
  const double tb = block_sum<kThreads>(b);
  if (threadIdx.x == 0) {
    *oa = ta;
    *ob = tb;
  }
}

__global__ void k_diag_of(const double *vals, const int64_t *diag_pos, int64_t N, double *d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = diag_pos[i];
    d[i] = q >= 0 ? vals[q] : 0.0;
  }
}

__global__ void k_invert(double *d, int64_t N, int *err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (!(d[i] > 0.0)) atomicOr(err, ERRW_NONFINITE);
    d[i] = 1.0 / d[i];
  }
}

// Block Jacobi (jacobi = 2): the D x D diagonal block of every node from the CSR values (its
// columns are contiguous in each of the node's rows: entry (nD+i, nD+k) sits at
// diag_pos[nD+i] + k - i), inverted in closed form.  Dirichlet rows are identity rows with
// zero off-diagonal columns, so their blocks stay invertible.
template <int D>
__global__ void k_block_jacobi(const double *vals, const int64_t *diag_pos, int64_t n_nodes,
                               double *binv, int *err) {
  for (int64_t nd = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; nd < n_nodes;
       nd += (int64_t)gridDim.x * blockDim.x) {
    double B[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int64_t q = diag_pos[nd * D + i];
#pragma unroll
      for (int k = 0; k < D; ++k) B[i][k] = vals[q + k - i];
    }
    double C[D][D], det;
    if constexpr (D == 2) {
      C[0][0] = B[1][1]; C[0][1] = -B[0][1]; C[1][0] = -B[1][0]; C[1][1] = B[0][0];
      det = B[0][0] * B[1][1] - B[0][1] * B[1][0];
    } else {  // adjugate: C = adj(B), B^-1 = C / det
      C[0][0] = B[1][1] * B[2][2] - B[1][2] * B[2][1];
      C[0][1] = B[0][2] * B[2][1] - B[0][1] * B[2][2];
      C[0][2] = B[0][1] * B[1][2] - B[0][2] * B[1][1];
      C[1][0] = B[1][2] * B[2][0] - B[1][0] * B[2][2];
      C[1][1] = B[0][0] * B[2][2] - B[0][2] * B[2][0];
      C[1][2] = B[0][2] * B[1][0] - B[0][0] * B[1][2];
      C[2][0] = B[1][0] * B[2][1] - B[1][1] * B[2][0];
      C[2][1] = B[0][1] * B[2][0] - B[0][0] * B[2][1];
      C[2][2] = B[0][0] * B[1][1] - B[0][1] * B[1][0];
      det = B[0][0] * C[0][0] + B[0][1] * C[1][0] + B[0][2] * C[2][0];
    }
    if (!(det > 0.0)) atomicOr(err, ERRW_NONFINITE);  // SPD blocks have det > 0
    const double id = 1.0 / det;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int k = 0; k < D; ++k) binv[(nd * D + i) * D + k] = C[i][k] * id;
  }
}

// block-preconditioned CG steps (one thread per node): z = B^-1 r per node, partial r.r, r.z;
// start: p = z; update: x += alpha p, r -= alpha Ap first
template <int D, bool START>
__global__ void k_cg_block(const double *scal, int rz_slot, double *x, double *r, double *zv,
                           double *p, const double *Ap, const double *binv, int64_t n_nodes,
                           double *part_rr, double *part_rz) {
  const double alpha = START ? 0.0 : scal[rz_slot] / scal[S_PAP];
  double rr = 0.0, rz = 0.0;
  for (int64_t nd = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; nd < n_nodes;
       nd += (int64_t)gridDim.x * blockDim.x) {
    double rv[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const int64_t k = nd * D + i;
      if constexpr (START) {
        rv[i] = r[k];
      } else {
        x[k] = fma(alpha, p[k], x[k]);
        rv[i] = fma(-alpha, Ap[k], r[k]);
        r[k] = rv[i];
      }
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double zi = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) zi = fma(binv[(nd * D + i) * D + k], rv[k], zi);
      zv[nd * D + i] = zi;
      if constexpr (START) p[nd * D + i] = zi;
      rr = fma(rv[i], rv[i], rr);
      rz = fma(rv[i], zi, rz);
    }
  }
  const double a = block_sum<kThreads>(rr);
  const double b = block_sum<kThreads>(rz);
  if (threadIdx.x == 0) {
    part_rr[blockIdx.x] = a;
    part_rz[blockIdx.x] = b;
  }
}

__global__ void k_neg_copy(const double *a, double *b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = -a[i];
}

__global__ void k_add(double *a, const double *b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] += b[i];
}

static fem_status apply_op(Problem *p, int op, const double *z, const double *vals, const double *x,
                           double *y, cudaStream_t s, unsigned extra = 0) {
  if (op == 0) return run_hvp(p, z, x, y, FEM_APPLY_BC | (extra & FEM_LINEARIZED), s);
  return run_spmv(p, vals, x, y, s);
}

static fem_status read_scalars(Problem *p, int n, cudaStream_t s) {
  FEM_CUDA(cudaMemcpyAsync(p->h_scal, p->scal, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  return FEM_OK;
}

fem_status run_cg(Problem *p, const double *z, const double *vals, const double *b, double *x,
                  const fem_cg_opts *o, fem_cg_report *rep, cudaStream_t s) {
  const int64_t n = p->N;
  const bool jac = o->jacobi != 0, blk = o->jacobi == 2;
  const int every = o->check_every > 0 ? o->check_every : 1;
  const int D = p->dim;
  fem_status st = ensure(p->cgbuf, sizeof(double) * n * (jac ? (blk ? 4 + D : 5) : 3));
  if (st) return st;
  double *r = (double *)p->cgbuf.ptr, *pp = r + n, *Ap = pp + n;
  double *zv = jac ? Ap + n : r, *dinv = jac ? Ap + 2 * n : nullptr;
  const int nb = grid_for(n, kThreads, kReduceBlocks);
  double *part_a = p->partials, *part_b = p->partials + kReduceBlocks;
  const int64_t nn = p->n_nodes;
  const int nbb = grid_for(nn, kThreads, kReduceBlocks);
  if (blk) {
    if (D == 3) k_block_jacobi<3><<<grid_for(nn), kThreads, 0, s>>>(vals, p->diag_pos, nn, dinv, p->d_err);
    else k_block_jacobi<2><<<grid_for(nn), kThreads, 0, s>>>(vals, p->diag_pos, nn, dinv, p->d_err);
  } else if (jac) {  // multi-GPU: interface rows of the local CSR hold partial sums -> halo add
    k_diag_of<<<grid_for(n), kThreads, 0, s>>>(vals, p->diag_pos, n, dinv);
    if (p->size > 1) {
      st = halo_add(p, dinv, s);
      if (st) return st;
    }
    k_invert<<<grid_for(n), kThreads, 0, s>>>(dinv, n, p->d_err);
  }
  // r0 = b - A x0
  st = apply_op(p, o->op, z, vals, x, Ap, s, o->hvp_flags);
  if (st) return st;
  k_sub<<<grid_for(n), kThreads, 0, s>>>(b, Ap, r, n);
  const uint8_t *own = p->size > 1 ? p->owned : nullptr;
  if (blk) {
    if (D == 3) k_cg_block<3, true><<<nbb, kThreads, 0, s>>>(p->scal, 0, x, r, zv, pp, Ap, dinv, nn, part_a, part_b);
    else k_cg_block<2, true><<<nbb, kThreads, 0, s>>>(p->scal, 0, x, r, zv, pp, Ap, dinv, nn, part_a, part_b);
  } else {
    k_cg_start<<<nb, kThreads, 0, s>>>(r, dinv, zv, pp, n, part_a, part_b, own, p->dim);
  }
  k_final_sum2<<<1, kThreads, 0, s>>>(part_a, part_b, blk ? nbb : nb, p->scal + S_RR0, p->scal + S_RZ0);
  st = allreduce(p, p->scal + S_RZ0, 2, s);   // rz and rr
  if (st) return st;
  st = launch_dot(p, b, b, n, p->scal + S_BB, s);
  if (st) return st;
  FEM_LAUNCH_CHECK("cg start");
  st = read_scalars(p, 8, s);
  if (st) return st;
  st = read_error_word(p, s);
  if (st) return st;
  const double bn = std::sqrt(p->h_scal[S_BB]);
  const double tol = std::fmax(o->rtol * bn, o->atol);
  double rn = std::sqrt(p->h_scal[S_RR0]);
  rep->res0 = rn;
  rep->iters = 0;
  rep->converged = 0;
  int it = 0;
  fem_status result = FEM_OK;
  // one CG iteration on slot parity cur (rz / rr of the current residual live in slot cur)
  auto body = [&](int cur, cudaStream_t s) -> fem_status {
    fem_status sb = apply_op(p, o->op, z, vals, pp, Ap, s, o->hvp_flags);
    if (sb) return sb;
    sb = launch_dot(p, pp, Ap, n, p->scal + S_PAP, s);
    if (sb) return sb;
    if (blk) {
      if (D == 3) k_cg_block<3, false><<<nbb, kThreads, 0, s>>>(p->scal, S_RZ0 + 2 * cur, x, r, zv, pp, Ap, dinv, nn, part_a, part_b);
      else k_cg_block<2, false><<<nbb, kThreads, 0, s>>>(p->scal, S_RZ0 + 2 * cur, x, r, zv, pp, Ap, dinv, nn, part_a, part_b);
    } else {
      k_cg_update<<<nb, kThreads, 0, s>>>(p->scal, S_RZ0 + 2 * cur, x, r, zv, pp, Ap, dinv, n, part_a,
                                          part_b, own, p->dim);
    }
    const int nxt = 2 * (cur ^ 1);
    k_final_sum2<<<1, kThreads, 0, s>>>(part_a, part_b, blk ? nbb : nb, p->scal + S_RR0 + nxt,
                                        p->scal + S_RZ0 + nxt);
    sb = allreduce(p, p->scal + S_RZ0 + nxt, 2, s);   // rz and rr of the new residual
    if (sb) return sb;
    k_cg_dir<<<grid_for(n), kThreads, 0, s>>>(p->scal, S_RZ0 + 2 * cur, S_RZ0 + nxt, zv, pp, n);
    FEM_LAUNCH_CHECK("cg iteration");
    return FEM_OK;
  };
  // Between host checks the iterations run as a CUDA graph of two iterations (the slot
  // parity pattern repeats every 2), captured once per solve: ~10 kernel launches per
  // iteration become one graph launch per pair (small problems are launch-bound).  On a
  // multi-GPU problem the NCCL all-reduces and the halo exchange (forked onto the comm
  // stream and joined by events) are captured with the kernels; if the capture is refused
  // the iterations launch directly (FEM_NO_GRAPHS forces that).
  bool graphs = every >= 2 && !getenv("FEM_NO_GRAPHS");
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  while (true) {
    if (rn <= tol) { rep->converged = 1; break; }
    if (it >= o->max_iter) { result = FEM_ERR_NOT_CONVERGED; break; }
    const int todo = std::min(every - it % every, o->max_iter - it);  // until the next check
    if (graphs && !exec && (it & 1) == 0 && todo >= 2) {
      // captured on a private stream (the legacy default stream cannot capture)
      if (!p->cap_stream) FEM_CUDA(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
      FEM_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeRelaxed));
      fem_status sc = body(0, p->cap_stream);
      if (!sc) sc = body(1, p->cap_stream);
      cudaError_t ce = cudaStreamEndCapture(p->cap_stream, &graph);
      if (!sc && ce == cudaSuccess) ce = cudaGraphInstantiate(&exec, graph, 0);
      if (sc || ce != cudaSuccess) {
        if (p->size == 1) {
          if (sc) return sc;
          FEM_CUDA(ce);
        }
        (void)cudaGetLastError();  // multi-GPU: capture refused -> direct launches
        if (graph) cudaGraphDestroy(graph);
        graph = nullptr;
        exec = nullptr;
        graphs = false;
      }
    }
    if (exec && (it & 1) == 0 && todo >= 2) {
      for (int k = 0; k < todo / 2; ++k) FEM_CUDA(cudaGraphLaunch(exec, s));
      it += 2 * (todo / 2);
      if (todo & 1) {
        st = body(it & 1, s);
        if (st) return st;
        ++it;
      }
    } else {
      st = body(it & 1, s);
      if (st) return st;
      ++it;
    }
    if (it % every == 0 || it >= o->max_iter) {
      st = read_scalars(p, 8, s);
      if (st) return st;
      if (!(p->h_scal[S_PAP] > 0.0)) { result = FEM_ERR_CG_BREAKDOWN; break; }
      rn = std::sqrt(p->h_scal[S_RR0 + 2 * (it & 1)]);
      if (!std::isfinite(rn)) { result = FEM_ERR_NONFINITE; break; }
    }
  }
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  rep->iters = it;
  rep->res = rn;
  st = read_error_word(p, s);
  if (st) return st;
  if (result == FEM_ERR_CG_BREAKDOWN) set_error("CG breakdown: p^T A p <= 0");
  if (result == FEM_ERR_NOT_CONVERGED) set_error("CG: iteration cap reached");
  return result;
}

// ------------------------------------------------------------------ MINRES (f2)
// Saddle-point systems of the periodic Lagrangian are
// symmetric indefinite, so CG does not apply; MINRES (Paige & Saunders 1975) minimises
// ||b - A x||_2 over the Krylov space with the Lanczos three-term recurrence and Givens
// QR updates.  Unpreconditioned.  The scalar recurrence runs in one device thread
// (k_minres_scalars) so the host only reads the residual estimate every check_every
// iterations; the vector work is three fused kernels per iteration around the operator.
enum { M_ALFA = 8, M_BB2 = 9, M_OLDB = 10, M_BETA = 11, M_DBAR = 12, M_EPS = 13, M_PHIBAR = 14,
       M_CS = 15, M_SN = 16, M_PHI = 17, M_DENOM = 18, M_DELTA = 19, M_OLDEPS = 20,
       M_BETA1 = 21, M_BN = 22, M_NSLOTS = 24 };

__global__ void k_minres_init(double *scal) {
  const double beta1 = sqrt(scal[M_BB2]);
  scal[M_BETA1] = beta1;
  scal[M_OLDB] = 0.0;
  scal[M_BETA] = beta1;
  scal[M_DBAR] = 0.0;
  scal[M_EPS] = 0.0;
  scal[M_PHIBAR] = beta1;
  scal[M_CS] = -1.0;
  scal[M_SN] = 0.0;
}

// v = y / beta ; t -= (beta / oldb) r1 (it >= 1) done after the operator: t holds A v
__global__ void k_minres_scale(const double *scal, const double *y, double *v, int64_t n) {
  const double sc = scal[M_BETA] > 0.0 ? 1.0 / scal[M_BETA] : 0.0;  // 0: Krylov space exhausted
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = sc * y[i];
}

__global__ void k_minres_lanczos1(const double *scal, int first, double *t, const double *r1,
                                  int64_t n) {
  if (first || !(scal[M_OLDB] > 0.0)) return;
  const double c = scal[M_BETA] / scal[M_OLDB];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    t[i] = fma(-c, r1[i], t[i]);
}

__global__ void k_minres_lanczos2(const double *scal, double *t, const double *r2, int64_t n) {
  const double c = scal[M_BETA] > 0.0 ? scal[M_ALFA] / scal[M_BETA] : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    t[i] = fma(-c, r2[i], t[i]);
}

__global__ void k_minres_scalars(double *scal) {
  const double alfa = scal[M_ALFA];
  const double oldb = scal[M_BETA];
  const double beta = sqrt(fmax(scal[M_BB2], 0.0));
  const double cs = scal[M_CS], sn = scal[M_SN], dbar = scal[M_DBAR];
  const double oldeps = scal[M_EPS];
  const double delta = cs * dbar + sn * alfa;
  const double gbar = sn * dbar - cs * alfa;
  const double epsln = sn * beta;
  const double dbar2 = -cs * beta;
  double gamma = hypot(gbar, beta);
  if (gamma < 1e-300) gamma = 1e-300;
  const double cs2 = gbar / gamma, sn2 = beta / gamma;
  const double phi = cs2 * scal[M_PHIBAR];
  scal[M_PHIBAR] = sn2 * scal[M_PHIBAR];
  scal[M_OLDB] = oldb;
  scal[M_BETA] = beta;
  scal[M_OLDEPS] = oldeps;
  scal[M_DELTA] = delta;
  scal[M_EPS] = epsln;
  scal[M_DBAR] = dbar2;
  scal[M_CS] = cs2;
  scal[M_SN] = sn2;
  scal[M_PHI] = phi;
  scal[M_DENOM] = 1.0 / gamma;
}

// w = (v - oldeps w1 - delta w2) / gamma (w1, w2 after the shift w1 <- w2, w2 <- w; the new
// w goes to the buffer of the retired w1), x += phi w
__global__ void k_minres_update(const double *scal, const double *v, const double *w1,
                                const double *w2, double *wout, double *x, int64_t n) {
  const double oe = scal[M_OLDEPS], de = scal[M_DELTA], dn = scal[M_DENOM], phi = scal[M_PHI];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double wn = (v[i] - oe * w1[i] - de * w2[i]) * dn;
    wout[i] = wn;
    x[i] = fma(phi, wn, x[i]);
  }
}

fem_status run_minres(Problem *p, const double *z, const double *vals, const double *b, double *x,
                      const fem_cg_opts *o, fem_cg_report *rep, cudaStream_t s) {
  const int64_t n = p->N;
  const int every = o->check_every > 0 ? o->check_every : 1;
  fem_status st = ensure(p->cgbuf, sizeof(double) * n * 7);
  if (st) return st;
  double *B0 = (double *)p->cgbuf.ptr;
  double *V = B0, *R1 = B0 + n, *R2 = B0 + 2 * n, *T = B0 + 3 * n, *W = B0 + 4 * n,
         *W1 = B0 + 5 * n, *W2 = B0 + 6 * n;
  const int g = grid_for(n);
  double *sc = p->scal;
  // r1 = b - A x; y = r1 (= R2 at the loop head); beta1 = ||r1||
  st = apply_op(p, o->op, z, vals, x, T, s, o->hvp_flags);
  if (st) return st;
  k_sub<<<g, kThreads, 0, s>>>(b, T, R2, n);
  FEM_CUDA(cudaMemcpyAsync(R1, R2, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  FEM_CUDA(cudaMemsetAsync(W, 0, sizeof(double) * n, s));
  FEM_CUDA(cudaMemsetAsync(W1, 0, sizeof(double) * n, s));
  FEM_CUDA(cudaMemsetAsync(W2, 0, sizeof(double) * n, s));
  st = launch_dot(p, R2, R2, n, sc + M_BB2, s);
  if (st) return st;
  st = launch_dot(p, b, b, n, sc + M_BN, s);
  if (st) return st;
  k_minres_init<<<1, 1, 0, s>>>(sc);
  FEM_LAUNCH_CHECK("minres start");
  st = read_scalars(p, M_NSLOTS, s);
  if (st) return st;
  st = read_error_word(p, s);
  if (st) return st;
  const double tol = std::fmax(o->rtol * std::sqrt(p->h_scal[M_BN]), o->atol);
  double rn = p->h_scal[M_BETA1];
  rep->res0 = rn;
  rep->iters = 0;
  rep->converged = 0;
  int it = 0;
  fem_status result = FEM_OK;
  // y lives in R2 at the loop head (r2 = y after the previous iteration); w = W, w1/w2 rotate
  // one MINRES iteration; the Lanczos (r1, r2, t) and direction (w, w1, w2) buffers rotate
  // with period 3, so 3 iterations captured as a CUDA graph replay with consistent pointers
  auto body = [&](bool first, cudaStream_t s) -> fem_status {
    k_minres_scale<<<g, kThreads, 0, s>>>(sc, R2, V, n);
    fem_status sb = apply_op(p, o->op, z, vals, V, T, s, o->hvp_flags);
    if (sb) return sb;
    k_minres_lanczos1<<<g, kThreads, 0, s>>>(sc, first, T, R1, n);
    sb = launch_dot(p, V, T, n, sc + M_ALFA, s);
    if (sb) return sb;
    k_minres_lanczos2<<<g, kThreads, 0, s>>>(sc, T, R2, n);
    sb = launch_dot(p, T, T, n, sc + M_BB2, s);
    if (sb) return sb;
    k_minres_scalars<<<1, 1, 0, s>>>(sc);
    // w1 <- w2, w2 <- w, w <- new (into the retired w1 buffer)
    k_minres_update<<<g, kThreads, 0, s>>>(sc, V, W2, W, W1, x, n);
    {
      double *ow = W, *ow1 = W1, *ow2 = W2;
      W = ow1; W1 = ow2; W2 = ow;
    }
    // r1 <- r2, r2 <- t, t <- old r1
    double *oR1 = R1;
    R1 = R2; R2 = T; T = oR1;
    FEM_LAUNCH_CHECK("minres iteration");
    return FEM_OK;
  };
  const bool graphs = p->size == 1 && every >= 3 && !getenv("FEM_NO_GRAPHS");
  cudaGraphExec_t exec[3] = {nullptr, nullptr, nullptr};  // keyed by the rotation phase
  cudaGraph_t graph[3] = {nullptr, nullptr, nullptr};
  while (true) {
    if (rn <= tol) { rep->converged = 1; break; }
    if (it >= o->max_iter) { result = FEM_ERR_NOT_CONVERGED; break; }
    if (p->h_scal[M_BETA] == 0.0 && it > 0) { rep->converged = 1; break; }  // invariant space
    const int todo = std::min(every - it % every, o->max_iter - it);
    if (graphs && it >= 1 && todo >= 3) {
      const int ph = it % 3;
      if (!exec[ph]) {
        if (!p->cap_stream) FEM_CUDA(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
        FEM_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeRelaxed));
        fem_status sc3 = FEM_OK;
        for (int k = 0; k < 3 && !sc3; ++k) sc3 = body(false, p->cap_stream);
        cudaError_t ce = cudaStreamEndCapture(p->cap_stream, &graph[ph]);
        if (sc3) return sc3;
        FEM_CUDA(ce);
        FEM_CUDA(cudaGraphInstantiate(&exec[ph], graph[ph], 0));
      }
      for (int k = 0; k < todo / 3; ++k) FEM_CUDA(cudaGraphLaunch(exec[ph], s));
      it += 3 * (todo / 3);
    } else {
      st = body(it == 0, s);
      if (st) return st;
      ++it;
    }
    if (it % every == 0 || it >= o->max_iter) {
      st = read_scalars(p, M_NSLOTS, s);
      if (st) return st;
      rn = p->h_scal[M_PHIBAR];
      if (!std::isfinite(rn)) { result = FEM_ERR_NONFINITE; break; }
    }
  }
  for (int k = 0; k < 3; ++k) {
    if (exec[k]) cudaGraphExecDestroy(exec[k]);
    if (graph[k]) cudaGraphDestroy(graph[k]);
  }
  rep->iters = it;
  // true residual ||b - A x|| for the report
  st = apply_op(p, o->op, z, vals, x, T, s, o->hvp_flags);
  if (st) return st;
  k_sub<<<g, kThreads, 0, s>>>(b, T, T, n);
  st = launch_dot(p, T, T, n, sc + M_BB2, s);
  if (st) return st;
  st = read_scalars(p, M_NSLOTS, s);
  if (st) return st;
  rep->res = std::sqrt(p->h_scal[M_BB2]);
  st = read_error_word(p, s);
  if (st) return st;
  if (result == FEM_ERR_NOT_CONVERGED) set_error("MINRES: iteration cap reached");
  return result;
}

}  // namespace fem

using namespace fem;

extern "C" {

fem_status fem_cg_solve(fem_problem *h, const double *z, const double *vals, const double *b,
                        double *x, const fem_cg_opts *o, fem_cg_report *rep, fem_stream stream) {
  FEM_NVTX_RANGE("fem_cg_solve");
  FEM_ARG(h && b && x && o && rep, "fem_cg_solve: null argument");
  FEM_ARG(o->op == 0 || o->op == 1, "fem_cg_solve: op must be 0 (HVP) or 1 (CSR)");
  FEM_ARG(o->op == 1 || z, "fem_cg_solve: op 0 needs z");
  FEM_ARG(o->op == 0 || (vals && h->p.have_pattern), "fem_cg_solve: op 1 needs vals and a pattern");
  FEM_ARG(!o->jacobi || (o->op == 1 && h->p.n_mpc == 0), "fem_cg_solve: Jacobi needs op 1, no MPC");
  FEM_ARG(o->jacobi >= 0 && o->jacobi <= 2, "fem_cg_solve: jacobi must be 0, 1 or 2");
  FEM_ARG(o->jacobi != 2 || h->p.size == 1, "fem_cg_solve: block Jacobi is single-GPU");
  return run_cg(&h->p, z, vals, b, x, o, rep, (cudaStream_t)stream);
}

fem_status fem_minres_solve(fem_problem *h, const double *z, const double *vals, const double *b,
                            double *x, const fem_cg_opts *o, fem_cg_report *rep,
                            fem_stream stream) {
  FEM_NVTX_RANGE("fem_minres_solve");
  FEM_ARG(h && b && x && o && rep, "fem_minres_solve: null argument");
  FEM_ARG(o->op == 0 || o->op == 1, "fem_minres_solve: op must be 0 (HVP) or 1 (CSR)");
  FEM_ARG(o->op == 1 || z, "fem_minres_solve: op 0 needs z");
  FEM_ARG(o->op == 0 || (vals && h->p.have_pattern), "fem_minres_solve: op 1 needs vals and a pattern");
  FEM_ARG(!o->jacobi, "fem_minres_solve: unpreconditioned");
  return run_minres(&h->p, z, vals, b, x, o, rep, (cudaStream_t)stream);
}

fem_status fem_newton_solve(fem_problem *h, double *z, const fem_newton_opts *o,
                            fem_newton_report *rep, fem_stream stream) {
  FEM_NVTX_RANGE("fem_newton_solve");
  FEM_ARG(h && z && o && rep, "fem_newton_solve: null argument");
  FEM_ARG(o->forcing >= 0.0 && o->forcing <= 1.0, "fem_newton_solve: forcing must be in [0, 1]");
  Problem *p = &h->p;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = p->N;
  double *buf = nullptr;
  const bool csr = o->cg.op == 1;
  fem_status st;
  if (csr) {
    st = build_colors(p, s);
    if (st) return st;
  }
  // 2 vectors (+ the CSR values: 3.7 GB at cfg 3) in a problem-owned workspace, allocated by the
  // first solve and kept: a cudaMalloc / cudaFree of that size per solve cost 0.1-1.3 s of host
  // time (r02, cfg 3 CSR Newton wall times 2.8-4.2 s for the same 2,800 CG iterations), and a
  // pool allocation paid the pool's growth in the first CSR solve after other large buffers
  const size_t bytes = sizeof(double) * (2 * n + (csr ? p->nnz : 0));
  st = ensure(p->nwbuf, bytes);
  if (st) return st;
  buf = (double *)p->nwbuf.ptr;
  double *r = buf, *dz = buf + n, *vals = csr ? buf + 2 * n : nullptr;
  rep->iters = rep->cg_iters = rep->converged = 0;
  double r0 = 0.0, r_prev = 0.0, eta_prev = 0.0;
  fem_status result = FEM_OK;
  for (int it = 0;; ++it) {
    st = run_residual(p, z, r, FEM_APPLY_BC, s);
    if (st) { result = st; break; }
    st = launch_dot(p, r, r, n, p->scal + S_NRM, s);
    if (st) { result = st; break; }
    st = read_scalars(p, 8, s);
    if (st) { result = st; break; }
    st = read_error_word(p, s);
    if (st) { result = st; break; }
    const double nr = std::sqrt(p->h_scal[S_NRM]);
    if (it == 0) r0 = nr;
    rep->res = nr;
    rep->iters = it;
    if (nr <= std::fmax(o->atol, o->rtol * r0)) { rep->converged = 1; break; }
    if (!std::isfinite(nr)) { result = FEM_ERR_NONFINITE; break; }
    if (it >= o->max_iter) { result = FEM_ERR_NOT_CONVERGED; break; }
    k_neg_copy<<<grid_for(n), kThreads, 0, s>>>(r, r, n);
    FEM_CUDA(cudaMemsetAsync(dz, 0, sizeof(double) * n, s));
    if (csr) {
      st = run_assemble(p, z, vals, FEM_APPLY_BC, s);
      if (st) { result = st; break; }
    }
    fem_cg_report cr{};
    fem_cg_opts co = o->cg;
    if (o->forcing > 0.0) {
      // inexact Newton-Krylov (reading R16): Eisenstat-Walker choice 2 (alpha = 2)
      constexpr double kEtaMax = 0.1;
      const double g = o->forcing;
      double eta = kEtaMax;
      if (it > 0) {
        const double q = nr / r_prev;
        eta = std::fmin(kEtaMax, g * q * q);
        const double sg = g * eta_prev * eta_prev;  // safeguard against a premature drop
        if (sg > 0.1) eta = std::fmin(kEtaMax, std::fmax(eta, sg));
      }
      const double tau = std::fmax(o->atol, o->rtol * r0);
      eta = std::fmin(kEtaMax, std::fmax(eta, 0.5 * tau / nr));  // no over-solving of the last step
      eta = std::fmax(eta, o->cg.rtol);
      co.rtol = eta;
      eta_prev = eta;
    }
    r_prev = nr;
    // matrix-free CG on the linearized tangent (fem_linearize: the cached metric form; cfg 3
    // HVP 0.76 vs 0.94 ms recomputed); FEM_NEWTON_RECOMPUTE=1 recomputes the state per HVP
    if (!csr && p->material == FEM_NEO_HOOKEAN && !getenv("FEM_NEWTON_RECOMPUTE")) {
      st = run_linearize(p, z, s);
      if (st) { result = st; break; }
      co.hvp_flags |= FEM_LINEARIZED;
    }
    // the Lagrangian Hessian of an MPC problem is indefinite: MINRES instead of CG (f2)
    st = p->n_mpc ? run_minres(p, z, vals, r, dz, &co, &cr, s)
                  : run_cg(p, z, vals, r, dz, &co, &cr, s);
    rep->cg_iters += cr.iters;
    if (st) { result = st; break; }
    k_add<<<grid_for(n), kThreads, 0, s>>>(z, dz, n);
  }
  rep->res0 = r0;
  cudaStreamSynchronize(s);
  return result;
}

}  // extern "C"
