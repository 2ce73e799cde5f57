// fem_core.cu — problem lifetime, energy / residual / HVP (Eq. 1-3, Alg. 1).
//
// Element kernels: one thread per element, grid-stride, geometry recomputed from the
// coordinates in registers (the byte-minimal "R" dataflow of DESIGN.md §5), gather of the
// element's nodal values, hand-derived P / dP (element.cuh), fp64 atomic scatter-add
// (RED.E.ADD.F64 in L2) of the nodal forces — the transpose of Alg. 1's gather.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "element.cuh"
#include "fem_internal.cuh"

namespace fem {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

fem_status cuda_status(cudaError_t e, const char *what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? FEM_ERR_OUT_OF_MEMORY : FEM_ERR_CUDA;
}

static bool pool_disabled() {  // FEM_NO_POOL=1: plain cudaMalloc / cudaFree (A/B)
  static const bool off = getenv("FEM_NO_POOL") != nullptr;
  return off;
}

fem_status pool_alloc(void **ptr, size_t bytes, cudaStream_t s) {
  if (pool_disabled()) {
    FEM_CUDA(cudaMalloc(ptr, bytes > 0 ? bytes : 1));
    return FEM_OK;
  }
  static thread_local int configured = -1;  // device whose default pool was configured
  int dev = 0;
  FEM_CUDA(cudaGetDevice(&dev));
  if (configured != dev) {
    cudaMemPool_t pool;
    FEM_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = (uint64_t)16 << 30;  // kPoolKeep: retain up to 16 GiB of freed memory
    FEM_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    configured = dev;
  }
  FEM_CUDA(cudaMallocAsync(ptr, bytes > 0 ? bytes : 1, s));
  return FEM_OK;
}

void pool_free(void *ptr, cudaStream_t s) {
  if (!ptr) return;
  if (pool_disabled()) cudaFree(ptr);
  else cudaFreeAsync(ptr, s);
}

fem_status ensure(Workspace &w, size_t bytes) {
  if (w.bytes >= bytes) return FEM_OK;
  if (w.ptr) cudaFree(w.ptr);
  w.ptr = nullptr;
  w.bytes = 0;
  FEM_CUDA(cudaMalloc(&w.ptr, bytes));
  w.bytes = bytes;
  return FEM_OK;
}

fem_status read_error_word(Problem *p, cudaStream_t s) {
  int h = 0;
  FEM_CUDA(cudaMemcpyAsync(&h, p->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  if (h) FEM_CUDA(cudaMemsetAsync(p->d_err, 0, sizeof(int), s));
  if (h & ERRW_INVERTED) {
    set_error("neo-Hookean element with J = det F <= 0 (InvertedElement)");
    return FEM_ERR_INVERTED_ELEMENT;
  }
  if (h & ERRW_TOO_MANY_COLORS) {
    set_error("coloring needs more than FEM_MAX_COLORS colors");
    return FEM_ERR_TOO_MANY_COLORS;
  }
  if (h & ERRW_ADJ_OVERFLOW) {
    set_error("a node exceeds an adjacency capacity: more than kMaxNodeAdj = 128 distinct "
              "neighbours, or more than kRowMaxDeg = 256 incident elements (row-gather assembly)");
    return FEM_ERR_INVALID_ARG;
  }
  if (h & ERRW_NONFINITE) {
    set_error("non-finite value");
    return FEM_ERR_NONFINITE;
  }
  return FEM_OK;
}

// ------------------------------------------------------------------ element kernels
// k_elem: the plain one-thread-per-element form with element-level atomics.  Kept as the
// baseline the tile kernels (fem_tiles.cu) are measured against (FEM_BASELINE_SCATTER).

struct ElemArgs {
  const double *coords;
  const int32_t *conn;
  int64_t E;
  double lam, mu;
  const uint8_t *phase;
  const double *lam_tab, *mu_tab;
  const uint8_t *node_bc;  // non-null: mask v at Dirichlet DOFs (HVP with FEM_APPLY_BC)
  const double *u, *v;
  double *out;
  double *partials;
  int *err;
  const int32_t *list;  // COLORED: the elements of one color (caller ids)
  int64_t n_list;
};

template <int D>
__device__ __forceinline__ void load_conn(const int32_t *conn, int64_t e, int32_t (&nd)[D + 1]) {
  if constexpr (D == 3) {
    const int4 c = __ldg(reinterpret_cast<const int4 *>(conn) + e);
    nd[0] = c.x; nd[1] = c.y; nd[2] = c.z; nd[3] = c.w;
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) nd[a] = __ldg(conn + e * 3 + a);
  }
}

template <int D>
__device__ __forceinline__ void gather(const double *f, const int32_t (&nd)[D + 1],
                                       double (&x)[D + 1][D]) {
#pragma unroll
  for (int a = 0; a < D + 1; ++a)
#pragma unroll
    for (int i = 0; i < D; ++i) x[a][i] = __ldg(f + (int64_t)nd[a] * D + i);
}

// COLORED (FEM_COLORED_SCATTER): the elements of one color share no node, so each adds its
// nodal vectors with plain loads / stores (no atomics, no conflicts); colors run in order.
template <int D, int MAT, int OP, bool MASK, bool COLORED = false>
__global__ void __launch_bounds__(kThreads) k_elem(ElemArgs A) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n_items = COLORED ? A.n_list : A.E;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < n_items; it += stride) {
    const int64_t e = COLORED ? (int64_t)__ldg(A.list + it) : it;
    int32_t nd[D + 1];
    load_conn<D>(A.conn, e, nd);
    double x[D + 1][D], G[D + 1][D], vol;
    gather<D>(A.coords, nd, x);
    geometry<D>(x, G, vol);
    double lam = A.lam, mu = A.mu;
    if (A.phase) {
      const int ph = A.phase[e];
      lam = A.lam_tab[ph];
      mu = A.mu_tab[ph];
    }
    double H[D][D];
    if (OP != OP_HVP || MAT == FEM_NEO_HOOKEAN) {
      double u[D + 1][D];
      gather<D>(A.u, nd, u);
      field_gradient<D>(u, G, H);
    }
    if constexpr (OP == OP_ENERGY) {
      if constexpr (MAT == FEM_LINEAR_ELASTIC) {
        acc += vol * le_psi<D>(H, lam, mu);
      } else {
        NHState<D> s;
        if (!nh_state<D>(H, s)) { atomicOr(A.err, ERRW_INVERTED); continue; }
        acc += vol * nh_psi<D>(H, s, lam, mu);
      }
    } else {
      double S[D][D];
      if constexpr (OP == OP_RESIDUAL) {
        if constexpr (MAT == FEM_LINEAR_ELASTIC) {
          le_stress<D>(H, lam, mu, S);
        } else {
          NHState<D> s;
          if (!nh_state<D>(H, s)) { atomicOr(A.err, ERRW_INVERTED); continue; }
          nh_stress<D>(s, lam, mu, S);
        }
      } else {
        double v[D + 1][D], dH[D][D];
        gather<D>(A.v, nd, v);
        if constexpr (MASK) {
#pragma unroll
          for (int a = 0; a < D + 1; ++a) {
            const unsigned bc = __ldg(A.node_bc + nd[a]);
#pragma unroll
            for (int i = 0; i < D; ++i)
              if (bc & (1u << i)) v[a][i] = 0.0;
          }
        }
        field_gradient<D>(v, G, dH);
        if constexpr (MAT == FEM_LINEAR_ELASTIC) {
          le_stress<D>(dH, lam, mu, S);  // linear: dP = P(dH)
        } else {
          NHState<D> s;
          if (!nh_state<D>(H, s)) { atomicOr(A.err, ERRW_INVERTED); continue; }
          nh_dstress<D>(s, lam, mu, dH, S);
        }
      }
      double f[D + 1][D];
      nodal_from_stress<D>(S, G, vol, f);
#pragma unroll
      for (int a = 0; a < D + 1; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) {
          if constexpr (COLORED) A.out[(int64_t)nd[a] * D + i] += f[a][i];
          else atomicAdd(A.out + (int64_t)nd[a] * D + i, f[a][i]);
        }
    }
  }
  if constexpr (OP == OP_ENERGY) {
    const double t = block_sum<kThreads>(acc);
    if (threadIdx.x == 0) A.partials[blockIdx.x] = t;
  }
}

template <int OP, bool MASK, bool COLORED = false>
static fem_status launch_elem(Problem *p, const ElemArgs &a, int grid, cudaStream_t s) {
  if (p->n_elems == 0) return FEM_OK;
#define FEM_DISPATCH(D, M) k_elem<D, M, OP, MASK, COLORED><<<grid, kThreads, 0, s>>>(a)
  if (p->dim == 2) {
    if (p->material == FEM_LINEAR_ELASTIC) FEM_DISPATCH(2, FEM_LINEAR_ELASTIC);
    else FEM_DISPATCH(2, FEM_NEO_HOOKEAN);
  } else {
    if (p->material == FEM_LINEAR_ELASTIC) FEM_DISPATCH(3, FEM_LINEAR_ELASTIC);
    else FEM_DISPATCH(3, FEM_NEO_HOOKEAN);
  }
#undef FEM_DISPATCH
  FEM_LAUNCH_CHECK("element kernel");
  return FEM_OK;
}

static ElemArgs elem_args(Problem *p) {
  ElemArgs a{};
  a.coords = p->coords;
  a.conn = p->conn;
  a.E = p->n_elems;
  a.lam = p->lam;
  a.mu = p->mu;
  a.phase = p->phase;
  a.lam_tab = p->lam_tab;
  a.mu_tab = p->mu_tab;
  a.err = p->d_err;
  return a;
}

// ------------------------------------------------------------------ small vector kernels
// owned != null: only DOFs of nodes this rank owns (multi-GPU dots)
__global__ void k_partial_dot(const double *a, const double *b, int64_t n, double scale,
                              double *partials, const uint8_t *owned = nullptr, int dim = 1) {
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    if (!owned || owned[i / dim]) acc = fma(a[i], b[i], acc);
  const double t = block_sum<kThreads>(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = scale * t;
}

__global__ void k_final_sum(const double *partials, int64_t n, double *out) {
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += partials[i];
  const double t = block_sum<kThreads>(acc);
  if (threadIdx.x == 0) *out = t;
}

fem_status launch_dot(Problem *p, const double *a, const double *b, int64_t n, double *out,
                      cudaStream_t s) {
  const int nb = grid_for(n, kThreads, kReduceBlocks);
  k_partial_dot<<<nb, kThreads, 0, s>>>(a, b, n, 1.0, p->partials, p->size > 1 ? p->owned : nullptr, p->dim);
  k_final_sum<<<1, kThreads, 0, s>>>(p->partials, nb, out);
  FEM_LAUNCH_CHECK("dot");
  return allreduce(p, out, 1, s);  // no-op on one rank
}

// lambda_k * g_k(u) partial sums (energy), g_k = u[s] - u[m] - b
__global__ void k_mpc_energy(const double *z, const int32_t *s, const int32_t *m, const double *b,
                             int64_t nc, int64_t nu, double *partials) {
  double acc = 0.0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nc;
       k += (int64_t)gridDim.x * blockDim.x)
    acc += z[nu + k] * (z[s[k]] - z[m[k]] - b[k]);
  const double t = block_sum<kThreads>(acc);
  if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// residual: r_u += B^T lambda, r_lambda = B u - b ; HVP: y_u += B^T w_lambda, y_lambda = B w_u
// (w = v masked at Dirichlet DOFs when node_bc != null).  PAPER.md P:497-498, App. B.
__global__ void k_mpc_apply(const double *z, const int32_t *s, const int32_t *m, const double *b,
                            int64_t nc, int64_t nu, int dim, const uint8_t *node_bc,
                            double *out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nc;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t sk = s[k], mk = m[k];
    double zs = z[sk], zm = z[mk];
    if (node_bc) {
      if (node_bc[sk / dim] & (1u << (sk % dim))) zs = 0.0;
      if (node_bc[mk / dim] & (1u << (mk % dim))) zm = 0.0;
    }
    const double lk = z[nu + k];
    atomicAdd(out + sk, lk);
    atomicAdd(out + mk, -lk);
    out[nu + k] = b ? (zs - zm - b[k]) : (zs - zm);
  }
}

// owned != null (FEM_LOCAL_ONLY on a multi-GPU rank): DOF-wise terms only on owned DOFs, so
// that the later halo sum counts them once
__global__ void k_axpy(double *y, const double *x, double a, int64_t n,
                       const uint8_t *owned = nullptr, int dim = 1) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!owned || owned[i / dim]) y[i] = fma(a, x[i], y[i]);
}

// y[D] = src[D] (src = v for the HVP) or 0 (src = null, residual)
__global__ void k_bc_fix(double *y, const int32_t *dofs, int64_t nd, const double *src,
                         const uint8_t *owned = nullptr, int dim = 1) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nd;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = dofs[k];
    y[d] = (src && (!owned || owned[d / dim])) ? src[d] : 0.0;
  }
}

__global__ void k_set_dirichlet(double *z, const int32_t *dofs, const double *vals, int64_t nd) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nd;
       k += (int64_t)gridDim.x * blockDim.x)
    z[dofs[k]] = vals[k];
}

// node_bc byte per node: the thread of the first Dirichlet DOF of a node writes the byte.
__global__ void k_node_bc(const int32_t *dofs, int64_t nd, int dim, uint8_t *node_bc) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nd;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t node = dofs[k] / dim;
    if (k > 0 && dofs[k - 1] / dim == node) continue;
    unsigned bits = 0;
    for (int64_t q = k; q < nd && dofs[q] / dim == node; ++q) bits |= 1u << (dofs[q] % dim);
    node_bc[node] = (uint8_t)bits;
  }
}

// Validation: ids in range and detJ > 1e-14 (bbox diagonal)^d (reading C20).
template <int D>
__global__ void k_validate(const double *coords, const int32_t *conn, int64_t E, int64_t n_nodes,
                           int *bad) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    int32_t nd[D + 1];
    bool ok = true;
#pragma unroll
    for (int a = 0; a < D + 1; ++a) {
      nd[a] = conn[e * (D + 1) + a];
      ok = ok && nd[a] >= 0 && nd[a] < n_nodes;
    }
    if (!ok) { atomicOr(bad, 1); continue; }
    double x[D + 1][D], G[D + 1][D], vol;
    gather<D>(coords, nd, x);
    const double det = geometry<D>(x, G, vol);
    double d2 = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double lo = x[0][i], hi = x[0][i];
#pragma unroll
      for (int a = 1; a < D + 1; ++a) { lo = fmin(lo, x[a][i]); hi = fmax(hi, x[a][i]); }
      d2 += (hi - lo) * (hi - lo);
    }
    const double eps = (D == 2) ? 1e-14 * d2 : 1e-14 * d2 * sqrt(d2);
    if (!(det > eps)) atomicOr(bad, 2);
  }
}

__global__ void k_validate_dofs(const int32_t *dd, int64_t nd, const int32_t *ms,
                                const int32_t *mm, int64_t nc, int64_t nu, int *bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nd; k += stride) {
    if (dd[k] < 0 || dd[k] >= nu || (k > 0 && dd[k] <= dd[k - 1])) atomicOr(bad, 1);
  }
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nc; k += stride) {
    if (ms[k] < 0 || ms[k] >= nu || mm[k] < 0 || mm[k] >= nu || ms[k] == mm[k]) atomicOr(bad, 1);
  }
}

// ------------------------------------------------------------------ internal runners

// Element pass of the residual / HVP on a multi-GPU problem: tiles touching interface nodes,
// then (exchange of their partials on the comm stream) the interior tiles, then the combine;
// FEM_LOCAL_ONLY runs the same two passes without the exchange.  Single GPU: one pass.
static fem_status element_pass_halo(Problem *p, int op, const double *z, const double *v,
                                    double *y, bool bc, bool det, bool local_only,
                                    cudaStream_t s) {
  if (p->size <= 1 || det) {
    fem_status st = tile_pass(p, op, z, v, y, bc, det, nullptr, s);
    if (st) return st;
    return (p->size > 1 && !local_only) ? halo_add(p, y, s) : FEM_OK;
  }
  fem_status st = build_tile_lists(p, s);
  if (st) return st;
  st = tile_pass(p, op, z, v, y, bc, false, nullptr, s, 1);
  if (st) return st;
  if (!local_only) {
    st = halo_begin(p, y, s);
    if (st) return st;
  }
  st = tile_pass(p, op, z, v, y, bc, false, nullptr, s, 2);
  if (st) return st;
  return local_only ? FEM_OK : halo_end(p, y, s);
}

// Element coloring (FEM_COLORED_SCATTER): greedy in element-tile (Morton) order, each element
// takes the smallest color none of its nodes' earlier elements holds (per-node 128-bit color
// masks); a host pass over the connectivity at setup.  Colors >= the max node-element
// degree (24 for interior Kuhn nodes).
static fem_status build_elem_colors(Problem *p, cudaStream_t s) {
  if (p->ecolor_list || p->n_elems == 0) return FEM_OK;
  fem_status st = build_tiles(p, s);
  if (st) return st;
  const int nen = p->nen;
  const int64_t E = p->n_elems;
  std::vector<int32_t> conn((size_t)E * nen), perm((size_t)E);
  FEM_CUDA(cudaMemcpyAsync(conn.data(), p->conn, sizeof(int32_t) * conn.size(), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaMemcpyAsync(perm.data(), p->tiles.perm, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  std::vector<uint64_t> mask((size_t)p->n_nodes * 2, 0ull);
  std::vector<uint8_t> col((size_t)E);
  std::vector<int64_t> cnt(129, 0);
  int nc = 0;
  for (int64_t i = 0; i < E; ++i) {
    const int64_t e = perm[i];
    uint64_t m0 = 0, m1 = 0;
    for (int a = 0; a < nen; ++a) {
      const int64_t n = conn[e * nen + a];
      m0 |= mask[2 * n];
      m1 |= mask[2 * n + 1];
    }
    int c = ~m0 ? __builtin_ctzll(~m0) : (~m1 ? 64 + __builtin_ctzll(~m1) : 128);
    if (c >= 128) {
      set_error("FEM_COLORED_SCATTER: more than 128 element colors");
      return FEM_ERR_TOO_MANY_COLORS;
    }
    for (int a = 0; a < nen; ++a) mask[2 * conn[e * nen + a] + (c >> 6)] |= 1ull << (c & 63);
    col[i] = (uint8_t)c;
    ++cnt[c + 1];
    nc = std::max(nc, c + 1);
  }
  p->ecolor_off.assign(nc + 1, 0);
  for (int c = 0; c < nc; ++c) p->ecolor_off[c + 1] = p->ecolor_off[c] + cnt[c + 1];
  std::vector<int32_t> list((size_t)E);
  std::vector<int64_t> fill(p->ecolor_off.begin(), p->ecolor_off.end() - 1);
  for (int64_t i = 0; i < E; ++i) list[fill[col[i]]++] = perm[i];
  FEM_CUDA(cudaMalloc(&p->ecolor_list, sizeof(int32_t) * E));
  FEM_CUDA(cudaMemcpyAsync(p->ecolor_list, list.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  return FEM_OK;
}

template <int OP, bool MASK>
static fem_status colored_pass(Problem *p, ElemArgs a, cudaStream_t s) {
  fem_status st = build_elem_colors(p, s);
  if (st) return st;
  for (size_t c = 0; c + 1 < p->ecolor_off.size(); ++c) {
    a.list = p->ecolor_list + p->ecolor_off[c];
    a.n_list = p->ecolor_off[c + 1] - p->ecolor_off[c];
    st = launch_elem<OP, MASK, true>(p, a, grid_for(a.n_list), s);
    if (st) return st;
  }
  return FEM_OK;
}

fem_status run_residual(Problem *p, const double *z, double *r, unsigned flags, cudaStream_t s) {
  const bool det = flags & FEM_DETERMINISTIC;
  if (!det || p->n_elems == 0) FEM_CUDA(cudaMemsetAsync(r, 0, sizeof(double) * p->N, s));
  fem_status st;
  if (flags & FEM_TILE_COLORED) {
    st = tile_pass(p, OP_RESIDUAL, z, nullptr, r, false, false, nullptr, s, 3);
  } else if (flags & FEM_COLORED_SCATTER) {
    ElemArgs a = elem_args(p);
    a.u = z;
    a.out = r;
    st = colored_pass<OP_RESIDUAL, false>(p, a, s);
  } else if (flags & FEM_BASELINE_SCATTER) {
    ElemArgs a = elem_args(p);
    a.u = z;
    a.out = r;
    st = launch_elem<OP_RESIDUAL, false>(p, a, grid_for(p->n_elems), s);
  } else {
    if (det && p->n_mpc) FEM_CUDA(cudaMemsetAsync(r + p->n_u, 0, sizeof(double) * p->n_mpc, s));
    const bool sg = flags & FEM_STREAM_GEOM;
    if (sg && det) {
      set_error("fem_residual: FEM_STREAM_GEOM with FEM_DETERMINISTIC");
      return FEM_ERR_INVALID_ARG;
    }
    const int op = sg ? OP_RESIDUAL_S : (flags & FEM_REFERENCE_METRIC) ? OP_RESIDUAL_R : OP_RESIDUAL;
    st = element_pass_halo(p, op, z, nullptr, r, false, det,
                           flags & FEM_LOCAL_ONLY, s);
  }
  if (st) return st;
  if ((flags & (FEM_BASELINE_SCATTER | FEM_COLORED_SCATTER | FEM_TILE_COLORED)) && p->size > 1 &&
      !(flags & FEM_LOCAL_ONLY)) {
    st = halo_add(p, r, s);
    if (st) return st;
  }
  return run_residual_terms(p, z, r, flags, s);
}

// the DOF-wise terms of the residual after the element pass: B^T lambda and g(u) (MPC),
// -f_ext, the Dirichlet rows
fem_status run_residual_terms(Problem *p, const double *z, double *r, unsigned flags,
                              cudaStream_t s) {
  if (p->n_mpc) {
    k_mpc_apply<<<grid_for(p->n_mpc), kThreads, 0, s>>>(z, p->mpc_s, p->mpc_m, p->mpc_b, p->n_mpc,
                                                        p->n_u, p->dim, nullptr, r);
  }
  const uint8_t *own = (p->size > 1 && (flags & FEM_LOCAL_ONLY)) ? p->owned : nullptr;
  if (p->f_ext) k_axpy<<<grid_for(p->n_u), kThreads, 0, s>>>(r, p->f_ext, -1.0, p->n_u, own, p->dim);
  if ((flags & FEM_APPLY_BC) && p->n_dir)
    k_bc_fix<<<grid_for(p->n_dir), kThreads, 0, s>>>(r, p->dir_dofs, p->n_dir, nullptr, own, p->dim);
  FEM_LAUNCH_CHECK("residual");
  return FEM_OK;
}

fem_status run_hvp(Problem *p, const double *z, const double *v, double *y, unsigned flags,
                   cudaStream_t s) {
  const bool det = flags & FEM_DETERMINISTIC;
  if (!det || p->n_elems == 0) FEM_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * p->N, s));
  const bool bc = (flags & FEM_APPLY_BC) && p->n_dir;
  fem_status st;
  if (flags & FEM_TILE_COLORED) {
    st = tile_pass(p, OP_HVP, z, v, y, bc, false, nullptr, s, 3);
  } else if (flags & FEM_COLORED_SCATTER) {
    ElemArgs a = elem_args(p);
    a.u = z;
    a.v = v;
    a.out = y;
    a.node_bc = p->node_bc;
    st = bc ? colored_pass<OP_HVP, true>(p, a, s) : colored_pass<OP_HVP, false>(p, a, s);
  } else if (flags & FEM_BASELINE_SCATTER) {
    ElemArgs a = elem_args(p);
    a.u = z;
    a.v = v;
    a.out = y;
    a.node_bc = p->node_bc;
    st = bc ? launch_elem<OP_HVP, true>(p, a, grid_for(p->n_elems), s)
            : launch_elem<OP_HVP, false>(p, a, grid_for(p->n_elems), s);
  } else {
    if (det && p->n_mpc) FEM_CUDA(cudaMemsetAsync(y + p->n_u, 0, sizeof(double) * p->n_mpc, s));
    const bool lin = (flags & FEM_LINEARIZED) && p->material == FEM_NEO_HOOKEAN;
    if (lin && !p->lin_valid) {
      set_error("fem_hvp: FEM_LINEARIZED without a preceding fem_linearize");
      return FEM_ERR_INVALID_ARG;
    }
    const bool sg = flags & FEM_STREAM_GEOM;
    if (sg && (det || lin)) {
      set_error("fem_hvp: FEM_STREAM_GEOM with FEM_DETERMINISTIC / FEM_LINEARIZED");
      return FEM_ERR_INVALID_ARG;
    }
    const int op = lin ? OP_HVP_LIN : sg ? OP_HVP_S : (flags & FEM_REFERENCE_METRIC) ? OP_HVP_R : OP_HVP;
    st = element_pass_halo(p, op, z, v, y, bc, det,
                           flags & FEM_LOCAL_ONLY, s);
  }
  if (st) return st;
  if ((flags & (FEM_BASELINE_SCATTER | FEM_COLORED_SCATTER | FEM_TILE_COLORED)) && p->size > 1 &&
      !(flags & FEM_LOCAL_ONLY)) {
    st = halo_add(p, y, s);
    if (st) return st;
  }
  if (p->n_mpc)
    k_mpc_apply<<<grid_for(p->n_mpc), kThreads, 0, s>>>(v, p->mpc_s, p->mpc_m, nullptr, p->n_mpc,
                                                        p->n_u, p->dim, bc ? p->node_bc : nullptr,
                                                        y);
  const uint8_t *own = (p->size > 1 && (flags & FEM_LOCAL_ONLY)) ? p->owned : nullptr;
  if (bc) k_bc_fix<<<grid_for(p->n_dir), kThreads, 0, s>>>(y, p->dir_dofs, p->n_dir, v, own, p->dim);
  FEM_LAUNCH_CHECK("hvp");
  return FEM_OK;
}

fem_status run_linearize(Problem *p, const double *z, cudaStream_t s) {
  if (p->material != FEM_NEO_HOOKEAN || p->n_elems == 0) {  // LE: the tangent is constant
    p->lin_valid = true;
    return FEM_OK;
  }
  fem_status st = build_tiles(p, s);
  if (st) return st;
  const int W = p->dim == 3 ? 3 * 3 + 2 + 6 : 2 * 2 + 2 + 3;   // lin_words(D), fem_tiles.cu
  if (!p->lin) FEM_CUDA(cudaMalloc(&p->lin, sizeof(double) * W * (size_t)p->tiles.n_tiles * kTile));
  st = tile_pass(p, OP_LIN, z, nullptr, nullptr, false, false, nullptr, s);
  if (st) return st;
  p->lin_valid = true;
  return FEM_OK;
}

}  // namespace fem

using namespace fem;

// ====================================================================== C ABI
// ------------------------------------------------------------------ mean stress (f2)
// Macroscopic stress of homogenization: the volume average of P(H_e) over the
// elements, per-block partials of (vol P, vol) in a fixed grid, then a fixed-order sum.
template <int D, int MAT>
__global__ void __launch_bounds__(kThreads) k_mean_stress(const double *coords, const int32_t *conn,
                                                         int64_t E, double lam0, double mu0,
                                                         const uint8_t *phase,
                                                         const double *lam_tab,
                                                         const double *mu_tab, const double *z,
                                                         double *partials, int *err) {
  constexpr int NEN = D + 1, Q = D * D + 1;
  double acc[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) acc[q] = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    double x[NEN][D], u[NEN][D], G[NEN][D], H[D][D], P[D][D], vol;
#pragma unroll
    for (int a = 0; a < NEN; ++a) {
      const int64_t n = conn[e * NEN + a];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        x[a][i] = coords[n * D + i];
        u[a][i] = z[n * D + i];
      }
    }
    geometry<D>(x, G, vol);
    field_gradient<D>(u, G, H);
    double lam = lam0, mu = mu0;
    if (phase) {
      lam = lam_tab[phase[e]];
      mu = mu_tab[phase[e]];
    }
    if constexpr (MAT == FEM_LINEAR_ELASTIC) {
      le_stress<D>(H, lam, mu, P);
    } else {
      NHState<D> st;
      if (!nh_state<D>(H, st)) {
        atomicOr(err, ERRW_INVERTED);
        continue;
      }
      nh_stress<D>(st, lam, mu, P);
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) acc[i * D + j] = fma(vol, P[i][j], acc[i * D + j]);
    acc[D * D] += vol;
  }
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const double t = block_sum<kThreads>(acc[q]);
    if (threadIdx.x == 0) partials[(int64_t)q * gridDim.x + blockIdx.x] = t;
  }
}

// ------------------------------------------------------------------ external loads (f3)
// Traction and body-force terms of the total potential energy (§6.1 Eq. P:366-372,
// listing P:380-386): Psi -= int_St t . u dGamma + int_Omega b . u dOmega.  Both are linear in
// u, so with P1 shape functions and a load constant per boundary facet / element they are
// exactly the consistent nodal loads int N_a t = t |facet| / n_facet_nodes (one-point rule
// of the Line2 / Tri3 boundary operator, exact here) and int N_a b = b vol / (d+1); they are
// accumulated into the problem's f_ext, which the energy, residual and Newton already use.
template <int D>
__global__ void k_traction_load(const double *coords, const int32_t *facets, int64_t nf,
                                const double *t, int64_t n_nodes, double *f, int *err) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nf;
       q += (int64_t)gridDim.x * blockDim.x) {
    int32_t nd[D];
    bool okid = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      nd[a] = facets[q * D + a];
      okid = okid && nd[a] >= 0 && nd[a] < n_nodes;
    }
    if (!okid) { atomicOr(err, ERRW_ADJ_OVERFLOW); continue; }
    double area;
    if constexpr (D == 2) {  // Line2: length
      const double dx = coords[nd[1] * 2] - coords[nd[0] * 2];
      const double dy = coords[nd[1] * 2 + 1] - coords[nd[0] * 2 + 1];
      area = sqrt(dx * dx + dy * dy);
    } else {                 // Tri3: half the cross-product norm
      double e1[3], e2[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        e1[i] = coords[nd[1] * 3 + i] - coords[nd[0] * 3 + i];
        e2[i] = coords[nd[2] * 3 + i] - coords[nd[0] * 3 + i];
      }
      const double cx = e1[1] * e2[2] - e1[2] * e2[1], cy = e1[2] * e2[0] - e1[0] * e2[2],
                   cz = e1[0] * e2[1] - e1[1] * e2[0];
      area = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
    }
    const double w = area / D;  // int N_a over the facet
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int i = 0; i < D; ++i) atomicAdd(f + (int64_t)nd[a] * D + i, w * t[q * D + i]);
  }
}

template <int D>
__global__ void k_body_load(const double *coords, const int32_t *conn, int64_t E, double b0,
                            double b1, double b2, double *f) {
  const double b[3] = {b0, b1, b2};
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    double x[D + 1][D], G[D + 1][D], vol;
#pragma unroll
    for (int a = 0; a < D + 1; ++a)
#pragma unroll
      for (int i = 0; i < D; ++i) x[a][i] = coords[(int64_t)conn[e * (D + 1) + a] * D + i];
    geometry<D>(x, G, vol);
    const double w = vol / (D + 1);
#pragma unroll
    for (int a = 0; a < D + 1; ++a)
#pragma unroll
      for (int i = 0; i < D; ++i) atomicAdd(f + (int64_t)conn[e * (D + 1) + a] * D + i, w * b[i]);
  }
}

static fem_status ensure_fext(Problem *p, cudaStream_t s) {
  if (p->f_ext) return FEM_OK;
  FEM_CUDA(cudaMalloc(&p->f_ext, sizeof(double) * (p->n_u > 0 ? p->n_u : 1)));
  FEM_CUDA(cudaMemsetAsync(p->f_ext, 0, sizeof(double) * (p->n_u > 0 ? p->n_u : 1), s));
  return FEM_OK;
}

extern "C" {

const char *fem_last_error(void) { return g_last_error.c_str(); }
const char *fem_version(void) { return "fem-b200 0.1 (sm_100a)"; }

fem_status fem_create(fem_problem **out, const fem_mesh_desc *d, const fem_dist_desc *dist,
                      fem_stream stream) {
  FEM_NVTX_RANGE("fem_create");
  FEM_ARG(out && d, "fem_create: null argument");
  *out = nullptr;
  FEM_ARG(d->dim == 2 || d->dim == 3, "fem_create: dim must be 2 or 3");
  FEM_ARG(d->n_nodes > 0 && d->n_elems >= 0, "fem_create: bad sizes");
  FEM_ARG(d->coords && (d->conn || d->n_elems == 0), "fem_create: null coords/conn");
  FEM_ARG(d->material == FEM_LINEAR_ELASTIC || d->material == FEM_NEO_HOOKEAN,
          "fem_create: unknown material");
  FEM_ARG(d->n_dirichlet >= 0 && (d->n_dirichlet == 0 || (d->dirichlet_dofs && d->dirichlet_vals)),
          "fem_create: bad Dirichlet arrays");
  FEM_ARG(d->n_mpc >= 0 && (d->n_mpc == 0 || (d->mpc_slave && d->mpc_master && d->mpc_offset)),
          "fem_create: bad MPC arrays");
  FEM_ARG(!d->phase || (d->lambda_tab && d->mu_tab && d->n_phases > 0 && d->n_phases <= 256),
          "fem_create: bad phase tables");
  FEM_ARG(d->n_nodes * d->dim + d->n_mpc < (int64_t)INT32_MAX, "fem_create: N exceeds int32");
  FEM_ARG(d->n_elems < (int64_t)1 << 29, "fem_create: too many elements");
  FEM_ARG(!(dist && dist->size > 1 && d->n_mpc), "fem_create: MPC with >1 rank unsupported");
  cudaStream_t s = (cudaStream_t)stream;
  fem_problem *h = new fem_problem();
  Problem *p = &h->p;
  p->dim = d->dim;
  p->nen = d->dim + 1;
  p->material = d->material;
  p->n_nodes = d->n_nodes;
  p->n_elems = d->n_elems;
  p->n_u = d->n_nodes * d->dim;
  p->n_mpc = d->n_mpc;
  p->N = p->n_u + p->n_mpc;
  p->n_dir = d->n_dirichlet;
  p->lam = d->lambda;
  p->mu = d->mu;
  p->n_phases = d->phase ? d->n_phases : 0;
  auto fail = [&](fem_status st) {
    fem_destroy(h);
    return st;
  };
#define FEM_C(call)                                   \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return fail(cuda_status(e_, #call)); \
  } while (0)
  const size_t cb = sizeof(double) * p->n_nodes * p->dim, nb = sizeof(int32_t) * p->n_elems * p->nen;
  FEM_C(cudaMalloc(&p->coords, cb));
  FEM_C(cudaMemcpyAsync(p->coords, d->coords, cb, cudaMemcpyDefault, s));
  FEM_C(cudaMalloc(&p->conn, nb > 0 ? nb : 16));
  if (nb) FEM_C(cudaMemcpyAsync(p->conn, d->conn, nb, cudaMemcpyDefault, s));
  if (d->phase) {
    FEM_C(cudaMalloc(&p->phase, p->n_elems > 0 ? p->n_elems : 1));
    if (p->n_elems) FEM_C(cudaMemcpyAsync(p->phase, d->phase, p->n_elems, cudaMemcpyDefault, s));
    FEM_C(cudaMalloc(&p->lam_tab, sizeof(double) * d->n_phases));
    FEM_C(cudaMalloc(&p->mu_tab, sizeof(double) * d->n_phases));
    FEM_C(cudaMemcpyAsync(p->lam_tab, d->lambda_tab, sizeof(double) * d->n_phases, cudaMemcpyDefault, s));
    FEM_C(cudaMemcpyAsync(p->mu_tab, d->mu_tab, sizeof(double) * d->n_phases, cudaMemcpyDefault, s));
  }
  FEM_C(cudaMalloc(&p->node_bc, p->n_nodes));
  FEM_C(cudaMemsetAsync(p->node_bc, 0, p->n_nodes, s));
  if (p->n_dir) {
    FEM_C(cudaMalloc(&p->dir_dofs, sizeof(int32_t) * p->n_dir));
    FEM_C(cudaMalloc(&p->dir_vals, sizeof(double) * p->n_dir));
    FEM_C(cudaMemcpyAsync(p->dir_dofs, d->dirichlet_dofs, sizeof(int32_t) * p->n_dir, cudaMemcpyDefault, s));
    FEM_C(cudaMemcpyAsync(p->dir_vals, d->dirichlet_vals, sizeof(double) * p->n_dir, cudaMemcpyDefault, s));
  }
  if (p->n_mpc) {
    FEM_C(cudaMalloc(&p->mpc_s, sizeof(int32_t) * p->n_mpc));
    FEM_C(cudaMalloc(&p->mpc_m, sizeof(int32_t) * p->n_mpc));
    FEM_C(cudaMalloc(&p->mpc_b, sizeof(double) * p->n_mpc));
    FEM_C(cudaMemcpyAsync(p->mpc_s, d->mpc_slave, sizeof(int32_t) * p->n_mpc, cudaMemcpyDefault, s));
    FEM_C(cudaMemcpyAsync(p->mpc_m, d->mpc_master, sizeof(int32_t) * p->n_mpc, cudaMemcpyDefault, s));
    FEM_C(cudaMemcpyAsync(p->mpc_b, d->mpc_offset, sizeof(double) * p->n_mpc, cudaMemcpyDefault, s));
  }
  if (d->f_ext) {
    FEM_C(cudaMalloc(&p->f_ext, sizeof(double) * p->n_u));
    FEM_C(cudaMemcpyAsync(p->f_ext, d->f_ext, sizeof(double) * p->n_u, cudaMemcpyDefault, s));
  }
  FEM_C(cudaMalloc(&p->partials, sizeof(double) * kReduceBlocks * 4));
  FEM_C(cudaMalloc(&p->scal, sizeof(double) * 64));
  FEM_C(cudaMemsetAsync(p->scal, 0, sizeof(double) * 64, s));
  FEM_C(cudaMallocHost(&p->h_scal, sizeof(double) * 64));
  FEM_C(cudaMalloc(&p->d_err, sizeof(int) * 2));
  FEM_C(cudaMemsetAsync(p->d_err, 0, sizeof(int) * 2, s));
  if (dist && dist->size > 1) {
    fem_status dst = dist_setup(p, dist, s);
    if (dst) return fail(dst);
  }
  // validation (ids, orientation / degeneracy, Dirichlet sortedness, MPC pairs)
  int *bad = p->d_err + 1;
  if (p->n_elems) {
    if (p->dim == 2)
      k_validate<2><<<grid_for(p->n_elems), kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->n_nodes, bad);
    else
      k_validate<3><<<grid_for(p->n_elems), kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->n_nodes, bad);
  }
  if (p->n_dir || p->n_mpc)
    k_validate_dofs<<<grid_for(p->n_dir > p->n_mpc ? p->n_dir : p->n_mpc), kThreads, 0, s>>>(
        p->dir_dofs, p->n_dir, p->mpc_s, p->mpc_m, p->n_mpc, p->n_u, bad);
  if (p->n_dir) k_node_bc<<<grid_for(p->n_dir), kThreads, 0, s>>>(p->dir_dofs, p->n_dir, p->dim, p->node_bc);
  FEM_C(cudaGetLastError());
  int hbad = 0;
  FEM_C(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  FEM_C(cudaStreamSynchronize(s));
  if (hbad & 1) {
    set_error("fem_create: index out of range / unsorted Dirichlet DOFs / invalid MPC pair");
    return fail(FEM_ERR_INVALID_ARG);
  }
  if (hbad & 2) {
    set_error("fem_create: degenerate or inverted element (detJ <= eps_det)");
    return fail(FEM_ERR_DEGENERATE_ELEMENT);
  }
#undef FEM_C
  fem_status tst = build_tiles(p, s);
  if (tst) return fail(tst);
  *out = h;
  return FEM_OK;
}

fem_status fem_destroy(fem_problem *h) {
  FEM_NVTX_RANGE("fem_destroy");
  if (!h) return FEM_OK;
  Problem *p = &h->p;
  // pattern / coloring buffers come from the stream-ordered pool (pool_alloc), for which
  // cudaFree does not synchronize: finish all work that may still read them first
  cudaDeviceSynchronize();
  void *bufs[] = {p->coords, p->conn, p->phase, p->lam_tab, p->mu_tab, p->node_bc, p->dir_dofs,
                  p->dir_vals, p->mpc_s, p->mpc_m, p->mpc_b, p->f_ext, p->partials, p->scal,
                  p->d_err, p->inc_ptr, p->inc, p->nadj_ptr, p->nadj, p->dmpc_ptr, p->dmpc,
                  p->row_ptr, p->col_idx, p->diag_pos, p->slot_list, p->slot_off, p->node_order, p->rp_node, p->epos, p->rp_ent, p->rt.meta, p->ct.meta, p->rp_soff, p->rp_sbc, p->colors, p->jcomp.ptr, p->cgbuf.ptr, p->slotbuf.ptr, p->ctxbuf.ptr, p->nwbuf.ptr,
                  p->tmp.ptr};
  for (void *b : bufs)
    if (b) cudaFree(b);
  if (p->h_scal) cudaFreeHost(p->h_scal);
  if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
  if (p->lin) cudaFree(p->lin);
  if (p->ecolor_list) cudaFree(p->ecolor_list);
  if (p->ncolor_list) cudaFree(p->ncolor_list);
  if (p->tslot) cudaFree(p->tslot);
  free_tiles(p->tiles);
  dist_free(p);
  delete h;
  return FEM_OK;
}

fem_status fem_query(const fem_problem *h, int64_t *n_total, int64_t *nnz, int32_t *n_colors) {
  FEM_ARG(h, "fem_query: null problem");
  const Problem *p = &h->p;
  if (n_total) *n_total = p->N;
  if (nnz) *nnz = p->have_pattern ? p->nnz : -1;
  if (n_colors) *n_colors = p->have_colors ? p->n_colors : -1;
  return FEM_OK;
}

fem_status fem_check(fem_problem *h, fem_stream stream) {
  FEM_NVTX_RANGE("fem_check");
  FEM_ARG(h, "fem_check: null problem");
  FEM_CUDA(cudaGetLastError());
  return read_error_word(&h->p, (cudaStream_t)stream);
}

fem_status fem_apply_dirichlet(fem_problem *h, double *z, fem_stream stream) {
  FEM_NVTX_RANGE("fem_apply_dirichlet");
  FEM_ARG(h && z, "fem_apply_dirichlet: null argument");
  Problem *p = &h->p;
  if (p->n_dir)
    k_set_dirichlet<<<grid_for(p->n_dir), kThreads, 0, (cudaStream_t)stream>>>(z, p->dir_dofs,
                                                                                p->dir_vals, p->n_dir);
  FEM_LAUNCH_CHECK("fem_apply_dirichlet");
  return FEM_OK;
}

// energy = sum of n_elem element-energy partials already in p->partials[0..n_elem) (0 or 1
// here: a single pre-summed value) + lambda . g(u) - f_ext . u, fixed-order final sum
static fem_status energy_finish(Problem *p, const double *z, double *energy, int n,
                                cudaStream_t s) {
  if (p->n_mpc) {
    const int g2 = grid_for(p->n_mpc, kThreads, kReduceBlocks);
    k_mpc_energy<<<g2, kThreads, 0, s>>>(z, p->mpc_s, p->mpc_m, p->mpc_b, p->n_mpc, p->n_u,
                                         p->partials + n);
    n += g2;
  }
  if (p->f_ext) {
    const int g3 = grid_for(p->n_u, kThreads, kReduceBlocks);
    k_partial_dot<<<g3, kThreads, 0, s>>>(p->f_ext, z, p->n_u, -1.0, p->partials + n,
                                          p->size > 1 ? p->owned : nullptr, p->dim);
    n += g3;
  }
  if (n == 0) FEM_CUDA(cudaMemsetAsync(energy, 0, sizeof(double), s));
  else k_final_sum<<<1, kThreads, 0, s>>>(p->partials, n, energy);
  FEM_LAUNCH_CHECK("energy");
  return allreduce(p, energy, 1, s);
}

fem_status fem_energy(fem_problem *h, const double *z, double *energy, fem_stream stream) {
  FEM_NVTX_RANGE("fem_energy");
  FEM_ARG(h && z && energy, "fem_energy: null argument");
  Problem *p = &h->p;
  cudaStream_t s = (cudaStream_t)stream;
  int n = 0;
  if (p->n_elems) {
    fem_status st = build_tiles(p, s);
    if (st) return st;
    st = tile_pass(p, OP_ENERGY, z, nullptr, nullptr, false, false, p->tiles.epart, s);
    if (st) return st;
    k_final_sum<<<1, kThreads, 0, s>>>(p->tiles.epart, tile_energy_partials(p), p->partials);
    n = 1;
  }
  return energy_finish(p, z, energy, n, s);
}

fem_status fem_energy_residual(fem_problem *h, const double *z, double *energy, double *r,
                               unsigned flags, fem_stream stream) {
  FEM_NVTX_RANGE("fem_energy_residual");
  FEM_ARG(h && z && energy && r, "fem_energy_residual: null argument");
  FEM_ARG(z != r, "fem_energy_residual: z and r alias");
  Problem *p = &h->p;
  cudaStream_t s = (cudaStream_t)stream;
  // one element pass on a single GPU with the default scatter; otherwise the two calls
  if (p->size > 1 || (flags & (FEM_DETERMINISTIC | FEM_BASELINE_SCATTER | FEM_STREAM_GEOM |
                                FEM_COLORED_SCATTER | FEM_TILE_COLORED)) || p->n_elems == 0) {
    fem_status st = fem_energy(h, z, energy, stream);
    if (st) return st;
    return run_residual(p, z, r, flags, s);
  }
  fem_status st = build_tiles(p, s);
  if (st) return st;
  FEM_CUDA(cudaMemsetAsync(r, 0, sizeof(double) * p->N, s));
  st = tile_pass(p, OP_RESIDUAL, z, nullptr, r, false, false, p->tiles.epart, s);
  if (st) return st;
  k_final_sum<<<1, kThreads, 0, s>>>(p->tiles.epart, tile_energy_partials(p, OP_RESIDUAL), p->partials);
  st = energy_finish(p, z, energy, 1, s);
  if (st) return st;
  return run_residual_terms(p, z, r, flags, s);
}

fem_status fem_residual(fem_problem *h, const double *z, double *r, unsigned flags,
                        fem_stream stream) {
  FEM_NVTX_RANGE("fem_residual");
  FEM_ARG(h && z && r, "fem_residual: null argument");
  FEM_ARG(z != r, "fem_residual: z and r alias");
  return run_residual(&h->p, z, r, flags, (cudaStream_t)stream);
}

fem_status fem_hvp(fem_problem *h, const double *z, const double *v, double *y, unsigned flags,
                   fem_stream stream) {
  FEM_NVTX_RANGE("fem_hvp");
  FEM_ARG(h && z && v && y, "fem_hvp: null argument");
  FEM_ARG(v != y && z != y, "fem_hvp: output aliases an input");
  return run_hvp(&h->p, z, v, y, flags, (cudaStream_t)stream);
}

fem_status fem_mean_stress(fem_problem *h, const double *z, double *sigma, double *volume,
                           fem_stream stream) {
  FEM_NVTX_RANGE("fem_mean_stress");
  FEM_ARG(h && z && sigma, "fem_mean_stress: null argument");
  Problem *p = &h->p;
  cudaStream_t s = (cudaStream_t)stream;
  const int D = p->dim, Q = D * D + 1;
  const int nb = kReduceBlocks;
  double *part = nullptr, *out = nullptr;
  FEM_CUDA(cudaMalloc(&part, sizeof(double) * (size_t)nb * Q));
  FEM_CUDA(cudaMalloc(&out, sizeof(double) * Q));
  if (p->n_elems == 0) FEM_CUDA(cudaMemsetAsync(part, 0, sizeof(double) * (size_t)nb * Q, s));
  else if (D == 2) {
    if (p->material == FEM_LINEAR_ELASTIC) k_mean_stress<2, FEM_LINEAR_ELASTIC><<<nb, kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, part, p->d_err);
    else k_mean_stress<2, FEM_NEO_HOOKEAN><<<nb, kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, part, p->d_err);
  } else {
    if (p->material == FEM_LINEAR_ELASTIC) k_mean_stress<3, FEM_LINEAR_ELASTIC><<<nb, kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, part, p->d_err);
    else k_mean_stress<3, FEM_NEO_HOOKEAN><<<nb, kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, part, p->d_err);
  }
  for (int q = 0; q < Q; ++q) k_final_sum<<<1, kThreads, 0, s>>>(part + (size_t)q * nb, nb, out + q);
  FEM_LAUNCH_CHECK("mean stress");
  fem_status st = FEM_OK;
  for (int q = 0; q < Q && !st; ++q) st = allreduce(p, out + q, 1, s);
  double h_out[10] = {0};
  if (!st) {
    FEM_CUDA(cudaMemcpyAsync(h_out, out, sizeof(double) * Q, cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaStreamSynchronize(s));
    st = read_error_word(p, s);
  }
  cudaFree(part);
  cudaFree(out);
  if (st) return st;
  const double V = h_out[D * D];
  for (int q = 0; q < D * D; ++q) sigma[q] = V > 0.0 ? h_out[q] / V : 0.0;
  if (volume) *volume = V;
  return FEM_OK;
}

fem_status fem_add_traction(fem_problem *h, int64_t n_facets, const int32_t *facets,
                            const double *traction, fem_stream stream) {
  FEM_NVTX_RANGE("fem_add_traction");
  FEM_ARG(h && n_facets >= 0, "fem_add_traction: bad arguments");
  FEM_ARG(n_facets == 0 || (facets && traction), "fem_add_traction: null facets / traction");
  Problem *p = &h->p;
  cudaStream_t s = (cudaStream_t)stream;
  if (n_facets == 0) return FEM_OK;
  fem_status st = ensure_fext(p, s);
  if (st) return st;
  double *tmp = nullptr;  // this rank's facet loads, summed over the ranks sharing a node
  FEM_CUDA(cudaMalloc(&tmp, sizeof(double) * (p->N > 0 ? p->N : 1)));
  FEM_CUDA(cudaMemsetAsync(tmp, 0, sizeof(double) * (p->N > 0 ? p->N : 1), s));
  const int g = grid_for(n_facets);
  if (p->dim == 2) k_traction_load<2><<<g, kThreads, 0, s>>>(p->coords, facets, n_facets, traction, p->n_nodes, tmp, p->d_err);
  else k_traction_load<3><<<g, kThreads, 0, s>>>(p->coords, facets, n_facets, traction, p->n_nodes, tmp, p->d_err);
  FEM_LAUNCH_CHECK("traction load");
  if (p->size > 1) st = halo_add(p, tmp, s);
  if (!st) k_axpy<<<grid_for(p->n_u), kThreads, 0, s>>>(p->f_ext, tmp, 1.0, p->n_u, nullptr, p->dim);
  FEM_CUDA(cudaStreamSynchronize(s));
  cudaFree(tmp);
  if (st) return st;
  int herr = 0;
  FEM_CUDA(cudaMemcpy(&herr, p->d_err, sizeof(int), cudaMemcpyDeviceToHost));
  if (herr & ERRW_ADJ_OVERFLOW) {
    FEM_CUDA(cudaMemset(p->d_err, 0, sizeof(int)));
    set_error("fem_add_traction: facet node id out of range");
    return FEM_ERR_INVALID_ARG;
  }
  return read_error_word(p, s);
}

fem_status fem_add_body_force(fem_problem *h, const double *b, fem_stream stream) {
  FEM_NVTX_RANGE("fem_add_body_force");
  FEM_ARG(h && b, "fem_add_body_force: null argument");
  Problem *p = &h->p;
  cudaStream_t s = (cudaStream_t)stream;
  fem_status st = ensure_fext(p, s);
  if (st) return st;
  double *tmp = nullptr;  // this rank's element loads, summed over the ranks sharing a node
  FEM_CUDA(cudaMalloc(&tmp, sizeof(double) * (p->N > 0 ? p->N : 1)));
  FEM_CUDA(cudaMemsetAsync(tmp, 0, sizeof(double) * (p->N > 0 ? p->N : 1), s));
  if (p->n_elems) {
    const int g = grid_for(p->n_elems);
    if (p->dim == 2) k_body_load<2><<<g, kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, b[0], b[1], 0.0, tmp);
    else k_body_load<3><<<g, kThreads, 0, s>>>(p->coords, p->conn, p->n_elems, b[0], b[1], b[2], tmp);
    FEM_LAUNCH_CHECK("body load");
  }
  if (p->size > 1) st = halo_add(p, tmp, s);
  if (!st) k_axpy<<<grid_for(p->n_u), kThreads, 0, s>>>(p->f_ext, tmp, 1.0, p->n_u, nullptr, p->dim);
  FEM_CUDA(cudaStreamSynchronize(s));
  cudaFree(tmp);
  return st;
}

fem_status fem_get_fext(fem_problem *h, double *f, fem_stream stream) {
  FEM_NVTX_RANGE("fem_get_fext");
  FEM_ARG(h && f, "fem_get_fext: null argument");
  Problem *p = &h->p;
  cudaStream_t s = (cudaStream_t)stream;
  if (p->f_ext) FEM_CUDA(cudaMemcpyAsync(f, p->f_ext, sizeof(double) * p->n_u, cudaMemcpyDeviceToDevice, s));
  else FEM_CUDA(cudaMemsetAsync(f, 0, sizeof(double) * p->n_u, s));
  return FEM_OK;
}

fem_status fem_linearize(fem_problem *h, const double *z, fem_stream stream) {
  FEM_NVTX_RANGE("fem_linearize");
  FEM_ARG(h && z, "fem_linearize: null argument");
  return run_linearize(&h->p, z, (cudaStream_t)stream);
}

}  // extern "C"
