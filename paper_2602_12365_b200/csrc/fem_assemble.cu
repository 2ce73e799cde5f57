// fem_assemble.cu — sparse tangent by Alg. 2 (a9 colored HVP -> J_comp, a10 decompression)
// and the CSR SpMV (a11).
//
// Element-Hessian columns.  The HVP along a unit seed e_(b,k) of element e is column (b,k)
// of the element tangent; with G_a the P1 gradients, g_a = F^{-T} G_a (spatial gradients),
// c1 = mu - lambda ln J (NH) / mu (LE), c2 = lambda and F = I for LE, it is
//   K_ab[i][k] = vol [ mu (G_a . G_b) delta_ik + c1 g_a[k] g_b[i] + c2 g_a[i] g_b[k] ],
// which is element.cuh's dP = mu dH + c1 F^{-T} dH^T F^{-T} + c2 (F^{-T}:dH) F^{-T} applied to
// dH = e_k (x) G_b and contracted with vol G_a (DESIGN.md §5 derives it).
#include <cuda_runtime.h>

#include "element.cuh"
#include "fem_internal.cuh"

namespace fem {

template <int D>
struct ColumnCtx {
  double G[D + 1][D];
  double g[D + 1][D];  // spatial gradients (== G for LE)
  double vol, mu, c1, c2;
};

// Builds the per-element context; false if the element is inverted (NH).
template <int D, int MAT>
__device__ __forceinline__ bool column_ctx(const double *coords, const int32_t (&nd)[D + 1],
                                           const double *z, double lam, double mu,
                                           ColumnCtx<D> &c) {
  double x[D + 1][D];
#pragma unroll
  for (int a = 0; a < D + 1; ++a)
#pragma unroll
    for (int i = 0; i < D; ++i) x[a][i] = __ldg(coords + (int64_t)nd[a] * D + i);
  geometry<D>(x, c.G, c.vol);
  c.mu = mu;
  c.c2 = lam;
  if constexpr (MAT == FEM_LINEAR_ELASTIC) {
    c.c1 = mu;
#pragma unroll
    for (int a = 0; a < D + 1; ++a)
#pragma unroll
      for (int i = 0; i < D; ++i) c.g[a][i] = c.G[a][i];
    return true;
  } else {
    double u[D + 1][D], H[D][D];
#pragma unroll
    for (int a = 0; a < D + 1; ++a)
#pragma unroll
      for (int i = 0; i < D; ++i) u[a][i] = __ldg(z + (int64_t)nd[a] * D + i);
    field_gradient<D>(u, c.G, H);
    NHState<D> s;
    if (!nh_state<D>(H, s)) return false;
    c.c1 = mu - lam * s.lnJ;
#pragma unroll
    for (int a = 0; a < D + 1; ++a)
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) t = fma(s.FiT[i][j], c.G[a][j], t);
        c.g[a][i] = t;
      }
    return true;
  }
}

// K_ab[i][k] for all i (column k of block ab)
template <int D>
__device__ __forceinline__ void column_block(const ColumnCtx<D> &c, int a, int b, int k,
                                             double (&out)[D]) {
  double GG = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) GG = fma(c.G[a][j], c.G[b][j], GG);
  const double ak = c.c1 * c.g[a][k], bk = c.c2 * c.g[b][k];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double t = fma(ak, c.g[b][i], bk * c.g[a][i]);
    if (i == k) t += c.mu * GG;
    out[i] = c.vol * t;
  }
}

struct AsmArgs {
  const double *coords;
  const int32_t *conn;
  int64_t E;
  double lam, mu;
  const uint8_t *phase;
  const double *lam_tab, *mu_tab;
  const uint8_t *node_bc;  // null: no masking
  const int32_t *colors;
  int C;
  const double *z;
  double *J;               // [N][C]
  int *err;
};

template <int D>
__device__ __forceinline__ void load_nodes(const int32_t *conn, int64_t e, int32_t (&nd)[D + 1]) {
  if constexpr (D == 3) {
    const int4 c = __ldg(reinterpret_cast<const int4 *>(conn) + e);
    nd[0] = c.x; nd[1] = c.y; nd[2] = c.z; nd[3] = c.w;
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) nd[a] = __ldg(conn + e * 3 + a);
  }
}

// All color passes in one element sweep: every element is active for the colors of its
// (dim+1)*dim DOFs and adds its response to J_comp[row][color(seed)].  LITERAL: only the
// seed of color `pass` (at most one per element).
template <int D, int MAT, bool LITERAL>
__global__ void __launch_bounds__(kThreads) k_colored_hvp(AsmArgs A, int pass) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < A.E; e += stride) {
    int32_t nd[D + 1];
    load_nodes<D>(A.conn, e, nd);
    int32_t col[D + 1][D];
    bool any = false;
#pragma unroll
    for (int b = 0; b < D + 1; ++b) {
      const unsigned bc = A.node_bc ? __ldg(A.node_bc + nd[b]) : 0u;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        int32_t c = __ldg(A.colors + (int64_t)nd[b] * D + k);
        if (bc & (1u << k)) c = -1;                // masked seed (P_f)
        if (LITERAL && c != pass) c = -1;
        col[b][k] = c;
        any = any || c >= 0;
      }
    }
    if (!any) continue;
    double lam = A.lam, mu = A.mu;
    if (A.phase) {
      const int ph = A.phase[e];
      lam = A.lam_tab[ph];
      mu = A.mu_tab[ph];
    }
    ColumnCtx<D> cx;
    if (!column_ctx<D, MAT>(A.coords, nd, A.z, lam, mu, cx)) {
      atomicOr(A.err, ERRW_INVERTED);
      continue;
    }
#pragma unroll
    for (int b = 0; b < D + 1; ++b)
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const int32_t c = col[b][k];
        if (c < 0) continue;
#pragma unroll
        for (int a = 0; a < D + 1; ++a) {
          double kab[D];
          column_block<D>(cx, a, b, k, kab);
#pragma unroll
          for (int i = 0; i < D; ++i)
            atomicAdd(A.J + ((int64_t)nd[a] * D + i) * A.C + c, kab[i]);
        }
      }
  }
}

// Multiplier rows of J_comp and the B^T columns: J[s_k][color(N_u+k)] += 1, J[m_k][..] -= 1;
// J[N_u+k][c] = [color(s_k)==c] (unmasked s_k) - [color(m_k)==c] (unmasked m_k).
__global__ void k_jcomp_mpc(const int32_t *ms, const int32_t *mm, int64_t nc, int64_t nu, int dim,
                            const uint8_t *node_bc, const int32_t *colors, int C, double *J) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nc;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = ms[k], m = mm[k];
    const int32_t cl = colors[nu + k];
    atomicAdd(J + (int64_t)s * C + cl, 1.0);
    atomicAdd(J + (int64_t)m * C + cl, -1.0);
    const bool ds = node_bc && (node_bc[s / dim] & (1u << (s % dim)));
    const bool dm = node_bc && (node_bc[m / dim] & (1u << (m % dim)));
    double *row = J + (nu + k) * C;
    for (int c = 0; c < C; ++c) row[c] = 0.0;
    if (!ds) row[colors[s]] += 1.0;
    if (!dm) row[colors[m]] -= 1.0;
  }
}

// Dirichlet rows of the masked operator: y[D] = e_c[D] for every color c.
__global__ void k_jcomp_bc(const int32_t *dofs, int64_t nd, const int32_t *colors, int C,
                           double *J) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nd;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = dofs[q];
    double *row = J + (int64_t)d * C;
    for (int c = 0; c < C; ++c) row[c] = (c == colors[d]) ? 1.0 : 0.0;
  }
}

// Alg. 2 part 2: K_ij = J_comp[i, color[j]] over the pattern (one thread per row).
__global__ void k_decompress(const int64_t *row_ptr, const int32_t *col_idx, const int32_t *colors,
                             const double *J, int C, int64_t N, double *vals) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N;
       r += (int64_t)gridDim.x * blockDim.x) {
    const double *jr = J + r * C;
    for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) vals[p] = jr[__ldg(colors + col_idx[p])];
  }
}

// ------------------------------------------------------------------ deterministic row gather
// One thread per node n: for its incident elements in ascending element order, the block
// row K_{a(n), b} is accumulated at the CSR slot of node b in n's sorted neighbour list
// (the compressed row of Alg. 2 stored at its decompressed positions), then written once.
constexpr int kRowMaxAdj = 32;

struct RowArgs {
  const double *coords;
  const int32_t *conn;
  double lam, mu;
  const uint8_t *phase;
  const double *lam_tab, *mu_tab;
  const uint8_t *node_bc;
  const double *z;
  const int64_t *inc_ptr;
  const int32_t *inc;
  const int64_t *nadj_ptr;
  const int32_t *nadj;
  const int32_t *dmpc_ptr, *dmpc, *ms, *mm;
  const int64_t *row_ptr;
  int64_t n_nodes, n_u;
  double *vals;
  int *err;
};

template <int D, int MAT>
__global__ void __launch_bounds__(128) k_rows_gather(RowArgs A) {
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < A.n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a0 = A.nadj_ptr[n];
    const int na = (int)(A.nadj_ptr[n + 1] - a0);
    if (na > kRowMaxAdj) { atomicOr(A.err, ERRW_ADJ_OVERFLOW); continue; }
    double acc[kRowMaxAdj][D][D];
    for (int q = 0; q < na; ++q)
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int k = 0; k < D; ++k) acc[q][i][k] = 0.0;
    const unsigned bcn = A.node_bc ? A.node_bc[n] : 0u;
    for (int64_t t = A.inc_ptr[n]; t < A.inc_ptr[n + 1]; ++t) {
      const int32_t packed = A.inc[t];
      const int64_t e = packed / (D + 1);
      const int a = packed % (D + 1);
      int32_t nd[D + 1];
      load_nodes<D>(A.conn, e, nd);
      double lam = A.lam, mu = A.mu;
      if (A.phase) {
        const int ph = A.phase[e];
        lam = A.lam_tab[ph];
        mu = A.mu_tab[ph];
      }
      ColumnCtx<D> cx;
      if (!column_ctx<D, MAT>(A.coords, nd, A.z, lam, mu, cx)) {
        atomicOr(A.err, ERRW_INVERTED);
        continue;
      }
#pragma unroll
      for (int b = 0; b < D + 1; ++b) {
        // slot of node nd[b] in n's sorted neighbour list
        int lo = 0, hi = na;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (A.nadj[a0 + mid] < nd[b]) lo = mid + 1; else hi = mid;
        }
        const unsigned bcb = A.node_bc ? __ldg(A.node_bc + nd[b]) : 0u;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          if (bcb & (1u << k)) continue;           // masked column
          double kab[D];
          column_block<D>(cx, a, b, k, kab);
#pragma unroll
          for (int i = 0; i < D; ++i) acc[lo][i][k] += kab[i];
        }
      }
    }
    for (int i = 0; i < D; ++i) {
      const int64_t r = n * D + i;
      const int64_t base = A.row_ptr[r];
      const bool drow = bcn & (1u << i);
      for (int q = 0; q < na; ++q)
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double v = acc[q][i][k];
          if (drow) v = (A.nadj[a0 + q] == n && k == i) ? 1.0 : 0.0;
          A.vals[base + q * D + k] = v;
        }
      if (A.dmpc_ptr) {  // B^T entries, ascending constraint id (same order as the pattern)
        const int32_t lo = A.dmpc_ptr[r], hi = A.dmpc_ptr[r + 1];
        int64_t w = base + (int64_t)na * D;
        int32_t prev = -1;
        for (int32_t q = lo; q < hi; ++q, ++w) {
          int32_t kmin = INT32_MAX;  // next constraint id above prev
          for (int32_t q2 = lo; q2 < hi; ++q2) {
            const int32_t kk = A.dmpc[q2];
            if (kk > prev && kk < kmin) kmin = kk;
          }
          prev = kmin;
          double v = (A.ms[kmin] == r ? 1.0 : 0.0) - (A.mm[kmin] == r ? 1.0 : 0.0);
          A.vals[w] = drow ? 0.0 : v;
        }
      }
    }
  }
}

__global__ void k_rows_mpc(const int32_t *ms, const int32_t *mm, int64_t nc, int64_t nu, int dim,
                           const uint8_t *node_bc, const int64_t *row_ptr, double *vals) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nc;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = ms[k], m = mm[k];
    const bool ds = node_bc && (node_bc[s / dim] & (1u << (s % dim)));
    const bool dm = node_bc && (node_bc[m / dim] & (1u << (m % dim)));
    const double vs = ds ? 0.0 : 1.0, vm = dm ? 0.0 : -1.0;
    const int64_t p = row_ptr[nu + k];
    vals[p] = s < m ? vs : vm;
    vals[p + 1] = s < m ? vm : vs;
  }
}

template <int D, int MAT>
static void launch_colored(const AsmArgs &a, bool literal, int pass, cudaStream_t s) {
  const int grid = grid_for(a.E);
  if (literal) k_colored_hvp<D, MAT, true><<<grid, kThreads, 0, s>>>(a, pass);
  else k_colored_hvp<D, MAT, false><<<grid, kThreads, 0, s>>>(a, pass);
}

static fem_status assemble(Problem *p, const double *z, double *vals, unsigned flags,
                           cudaStream_t s) {
  const bool bc = (flags & FEM_APPLY_BC) && p->n_dir;
  if (flags & FEM_DETERMINISTIC) {
    RowArgs A{};
    A.coords = p->coords; A.conn = p->conn; A.lam = p->lam; A.mu = p->mu;
    A.phase = p->phase; A.lam_tab = p->lam_tab; A.mu_tab = p->mu_tab;
    A.node_bc = bc ? p->node_bc : nullptr; A.z = z;
    A.inc_ptr = p->inc_ptr; A.inc = p->inc; A.nadj_ptr = p->nadj_ptr; A.nadj = p->nadj;
    A.dmpc_ptr = p->dmpc_ptr; A.dmpc = p->dmpc; A.ms = p->mpc_s; A.mm = p->mpc_m;
    A.row_ptr = p->row_ptr; A.n_nodes = p->n_nodes; A.n_u = p->n_u; A.vals = vals; A.err = p->d_err;
    const int grid = grid_for(p->n_nodes, 128);
    if (p->dim == 2) {
      if (p->material == FEM_LINEAR_ELASTIC) k_rows_gather<2, FEM_LINEAR_ELASTIC><<<grid, 128, 0, s>>>(A);
      else k_rows_gather<2, FEM_NEO_HOOKEAN><<<grid, 128, 0, s>>>(A);
    } else {
      if (p->material == FEM_LINEAR_ELASTIC) k_rows_gather<3, FEM_LINEAR_ELASTIC><<<grid, 128, 0, s>>>(A);
      else k_rows_gather<3, FEM_NEO_HOOKEAN><<<grid, 128, 0, s>>>(A);
    }
    if (p->n_mpc)
      k_rows_mpc<<<grid_for(p->n_mpc), kThreads, 0, s>>>(p->mpc_s, p->mpc_m, p->n_mpc, p->n_u, p->dim,
                                                         bc ? p->node_bc : nullptr, p->row_ptr, vals);
    FEM_LAUNCH_CHECK("row-gather assembly");
    return FEM_OK;
  }
  const int C = p->n_colors;
  fem_status st = ensure(p->jcomp, sizeof(double) * (size_t)p->N * C);
  if (st) return st;
  double *J = (double *)p->jcomp.ptr;
  FEM_CUDA(cudaMemsetAsync(J, 0, sizeof(double) * (size_t)p->N * C, s));
  AsmArgs a{};
  a.coords = p->coords; a.conn = p->conn; a.E = p->n_elems; a.lam = p->lam; a.mu = p->mu;
  a.phase = p->phase; a.lam_tab = p->lam_tab; a.mu_tab = p->mu_tab;
  a.node_bc = bc ? p->node_bc : nullptr; a.colors = p->colors; a.C = C; a.z = z; a.J = J;
  a.err = p->d_err;
  const bool literal = flags & FEM_ASSEMBLE_LITERAL;
  if (p->n_elems) {
    const int passes = literal ? C : 1;
    for (int c = 0; c < passes; ++c) {
      if (p->dim == 2) {
        if (p->material == FEM_LINEAR_ELASTIC) launch_colored<2, FEM_LINEAR_ELASTIC>(a, literal, c, s);
        else launch_colored<2, FEM_NEO_HOOKEAN>(a, literal, c, s);
      } else {
        if (p->material == FEM_LINEAR_ELASTIC) launch_colored<3, FEM_LINEAR_ELASTIC>(a, literal, c, s);
        else launch_colored<3, FEM_NEO_HOOKEAN>(a, literal, c, s);
      }
    }
  }
  if (p->n_mpc)
    k_jcomp_mpc<<<grid_for(p->n_mpc), kThreads, 0, s>>>(p->mpc_s, p->mpc_m, p->n_mpc, p->n_u, p->dim,
                                                        bc ? p->node_bc : nullptr, p->colors, C, J);
  if (bc) k_jcomp_bc<<<grid_for(p->n_dir), kThreads, 0, s>>>(p->dir_dofs, p->n_dir, p->colors, C, J);
  k_decompress<<<grid_for(p->N), kThreads, 0, s>>>(p->row_ptr, p->col_idx, p->colors, J, C, p->N, vals);
  FEM_LAUNCH_CHECK("colored assembly");
  return FEM_OK;
}

// ------------------------------------------------------------------ SpMV
template <int LPR>
__global__ void __launch_bounds__(256) k_spmv(const int64_t *row_ptr, const int32_t *col_idx,
                                              const double *vals, const double *x, double *y,
                                              int64_t N) {
  const int lane = threadIdx.x % LPR;
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x / LPR);
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR; r < N; r += groups) {
    const int64_t lo = row_ptr[r], hi = row_ptr[r + 1];
    double acc = 0.0;
    for (int64_t p = lo + lane; p < hi; p += LPR) acc = fma(__ldg(vals + p), __ldg(x + __ldg(col_idx + p)), acc);
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o, LPR);
    if (lane == 0) y[r] = acc;
  }
}

fem_status run_spmv(Problem *p, const double *vals, const double *x, double *y, cudaStream_t s) {
  const int64_t avg = p->N ? p->nnz / p->N : 0;
  const int64_t threads_needed = p->N * (avg > 24 ? 8 : 4);
  const int grid = grid_for(threads_needed, 256, 148 * 32);
  if (avg > 24) k_spmv<8><<<grid, 256, 0, s>>>(p->row_ptr, p->col_idx, vals, x, y, p->N);
  else k_spmv<4><<<grid, 256, 0, s>>>(p->row_ptr, p->col_idx, vals, x, y, p->N);
  FEM_LAUNCH_CHECK("spmv");
  if (p->size > 1) return halo_add(p, y, s);
  return FEM_OK;
}

fem_status run_assemble(Problem *p, const double *z, double *vals, unsigned flags, cudaStream_t s) {
  fem_status st = build_colors(p, s);
  if (st) return st;
  return assemble(p, z, vals, flags, s);
}

}  // namespace fem

using namespace fem;

extern "C" {

fem_status fem_assemble_csr(fem_problem *h, const double *z, double *vals, unsigned flags,
                            fem_stream stream) {
  FEM_ARG(h && z && vals, "fem_assemble_csr: null argument");
  return run_assemble(&h->p, z, vals, flags, (cudaStream_t)stream);
}

fem_status fem_spmv(fem_problem *h, const double *vals, const double *x, double *y,
                    fem_stream stream) {
  FEM_ARG(h && vals && x && y, "fem_spmv: null argument");
  FEM_ARG(h->p.have_pattern, "fem_spmv: call fem_sparsity first");
  FEM_ARG(x != y, "fem_spmv: x and y alias");
  return run_spmv(&h->p, vals, x, y, (cudaStream_t)stream);
}

}  // extern "C"
