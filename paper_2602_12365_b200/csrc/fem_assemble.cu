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

#include <cstdlib>

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
// 8 lanes per row: coalesced col_idx / vals streams, the row's J_comp entries (C doubles,
// contiguous) gathered through L1.
__global__ void k_decompress(const int64_t *row_ptr, const int32_t *col_idx, const int32_t *colors,
                             const double *J, int C, int64_t N, double *vals) {
  const int lane = threadIdx.x & 7;
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x / 8);
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 8; r < N; r += groups) {
    const double *jr = J + r * C;
    for (int64_t p = row_ptr[r] + lane; p < row_ptr[r + 1]; p += 8)
      vals[p] = __ldg(jr + __ldg(colors + __ldg(col_idx + p)));
  }
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ------------------------------------------------------------------ per-element tangent context
// k_elem_ctx evaluates, once per element, everything the element Hessian needs (the
// ColumnCtx above): per element node a = 0..d the pair (G_a, g_a), then the scalars vol*mu,
// vol*c1, vol*c2, stored as one 16-byte aligned record [G_0 g_0 | ... | G_d g_d | smu sc1
// sc2 pad].  The row-pull assembly then reads
// these records instead of re-gathering coordinates and state and re-evaluating F, F^-1
// and ln J for each of the element's nodes.

template <int D>
struct CtxLite {
  double G[D + 1][D], g[D + 1][D], smu, sc1, sc2;
};

template <int D>
__device__ __forceinline__ void load_ctx(const double *ctx, int64_t e, CtxLite<D> &c) {
  constexpr int ST = ctx_stride<D>();
  const double2 *p = reinterpret_cast<const double2 *>(ctx + e * ST);
  double v[ST];
#pragma unroll
  for (int q = 0; q < ST / 2; ++q) {
    const double2 t = p[q];
    v[2 * q] = t.x;
    v[2 * q + 1] = t.y;
  }
#pragma unroll
  for (int a = 0; a < D + 1; ++a)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      c.G[a][j] = v[a * 2 * D + j];
      c.g[a][j] = v[a * 2 * D + D + j];
    }
  c.smu = v[2 * D * (D + 1)];
  c.sc1 = v[2 * D * (D + 1) + 1];
  c.sc2 = v[2 * D * (D + 1) + 2];
}

constexpr int kCtxThreads = 128;

template <int D, int MAT>
__global__ void __launch_bounds__(kCtxThreads) k_elem_ctx(const double *coords, const int32_t *conn,
                                                         int64_t E, double lam0, double mu0,
                                                         const uint8_t *phase, const double *lam_tab,
                                                         const double *mu_tab, const double *z,
                                                         const int32_t *perm, double *ctx, int *err) {
  // record i holds element perm[i] (the element tiles' Morton order) or element i; each CTA
  // stages its kCtxThreads consecutive records in shared memory and stores them coalesced
  constexpr int ST = ctx_stride<D>();
  __shared__ __align__(16) double srec[kCtxThreads * ST];
  for (int64_t i0 = (int64_t)blockIdx.x * kCtxThreads; i0 < E; i0 += (int64_t)gridDim.x * kCtxThreads) {
    const int64_t i = i0 + threadIdx.x;
    if (i < E) {
      const int64_t e = perm ? (int64_t)__ldg(perm + i) : i;
      int32_t nd[D + 1];
      load_nodes<D>(conn, e, nd);
      double lam = lam0, mu = mu0;
      if (phase) {
        const int ph = phase[e];
        lam = lam_tab[ph];
        mu = mu_tab[ph];
      }
      ColumnCtx<D> cx;
      const bool ok = column_ctx<D, MAT>(coords, nd, z, lam, mu, cx);
      if (!ok) atomicOr(err, ERRW_INVERTED);
      double v[ST];
#pragma unroll
      for (int a = 0; a < D + 1; ++a)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          v[a * 2 * D + j] = ok ? cx.G[a][j] : 0.0;
          v[a * 2 * D + D + j] = ok ? cx.g[a][j] : 0.0;
        }
      constexpr int S0 = 2 * D * (D + 1);
      v[S0] = ok ? cx.vol * cx.mu : 0.0;
      v[S0 + 1] = ok ? cx.vol * cx.c1 : 0.0;
      v[S0 + 2] = ok ? cx.vol * cx.c2 : 0.0;
#pragma unroll
      for (int q = S0 + 3; q < ST; ++q) v[q] = 0.0;
      double2 *o = reinterpret_cast<double2 *>(srec + threadIdx.x * ST);
#pragma unroll
      for (int q = 0; q < ST / 2; ++q) o[q] = make_double2(v[2 * q], v[2 * q + 1]);
    }
    __syncthreads();
    const int64_t nrec = (E - i0 < kCtxThreads) ? E - i0 : kCtxThreads;
    const double2 *src = reinterpret_cast<const double2 *>(srec);
    double2 *dst = reinterpret_cast<double2 *>(ctx + i0 * ST);
    for (int q = threadIdx.x; q < nrec * (ST / 2); q += kCtxThreads) dst[q] = src[q];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ fused row-pull (deterministic)
// One warp per node n (32 lanes).  Lane l takes the l-th incident element of n (ascending
// element order), evaluates that element's column context once and its block row
// K_{a(n), b} for every element node b into shared memory.  Lane s then owns slot s of n's
// sorted neighbour list (i.e. the CSR columns of node nadj[s]) and sums, in a fixed
// precomputed order, the staged blocks that land on it: the compressed row of Alg. 2 at
// its decompressed positions (within a row every color names exactly one column, so the
// color -> CSR slot map is a bijection).  No atomics, bitwise reproducible, each value
// written once.  slot lists: per node, entries (l << 2 | b) grouped by slot (setup).
#ifndef FEM_ROWS_MINB
#define FEM_ROWS_MINB 4
#endif
constexpr int kRowLanes = 32;
constexpr int kRowGroups = 4;  // warps (nodes) per 128-thread CTA

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
  const uint16_t *slot_list;
  const uint16_t *slot_off;
  const int32_t *dmpc_ptr, *dmpc, *ms, *mm;
  const int64_t *row_ptr;
  const double *ctx;
  const int32_t *node_order;
  int64_t n_nodes, n_u;
  int dim;
  double *vals;
  int *err;
  const uint8_t *tslot;         // TR: position of n in the adjacency of its slot-s neighbour
};

template <int D>
__global__ void k_slot_build(const int64_t *inc_ptr, const int32_t *inc, const int32_t *conn,
                             const int64_t *nadj_ptr, const int32_t *nadj, int64_t n_nodes,
                             uint16_t *slot_list, uint16_t *slot_off, int *err) {
  constexpr int NEN = D + 1;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int deg = (int)(inc_ptr[n + 1] - inc_ptr[n]);
    const int64_t a0 = nadj_ptr[n];
    const int sn = (int)(nadj_ptr[n + 1] - a0);
    if (deg > kRowMaxDeg || sn > kMaxNodeAdj) { atomicOr(err, ERRW_ADJ_OVERFLOW); continue; }
    uint16_t cnt[kMaxNodeAdj + 1];
    for (int q = 0; q <= sn; ++q) cnt[q] = 0;
    for (int pass = 0; pass < 2; ++pass) {
      for (int l = 0; l < deg; ++l) {
        const int64_t e = inc[inc_ptr[n] + l] / NEN;
        for (int b = 0; b < NEN; ++b) {
          const int32_t m = conn[e * NEN + b];
          int lo = 0, hi = sn;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (nadj[a0 + mid] < m) lo = mid + 1; else hi = mid;
          }
          if (pass == 0) cnt[lo + 1]++;
          else slot_list[NEN * inc_ptr[n] + cnt[lo]++] = (uint16_t)(l << 2 | b);
        }
      }
      if (pass == 0) {
        for (int q = 0; q < sn; ++q) cnt[q + 1] += cnt[q];
        for (int q = 0; q <= sn; ++q) slot_off[a0 + n + q] = cnt[q];
      }
    }
  }
}

__device__ __forceinline__ int64_t rp_row(const RowArgs &A, int64_t n, int i) {
  return __ldg(A.row_ptr + n * (int64_t)A.dim + i);
}

// TR (FEM_ASSEMBLE_COLORED): the fused colored form of Alg. 2.  node_order lists the seed
// nodes of ONE node color; for seed n the warp evaluates K e_j for its D seed DOFs j (the
// columns n D + k) from the incident elements and writes each compressed entry directly at
// its decompressed CSR slot (row m D + i, column n D + k) — no J_comp.  Within a color no
// two seeds share a row (distance-2), and every (row, column) slot belongs to one seed, so
// the writes are conflict-free plain stores.  By the symmetry of every element Hessian the
// column block K[m, n] is the transpose of the row block the row form computes, so the same
// warp code produces it; only where it is written changes.
template <int D, bool TR = false>
__global__ void __launch_bounds__(kRowLanes * kRowGroups, FEM_ROWS_MINB) k_rows_fused(RowArgs A) {
  constexpr int NEN = D + 1, BS = D * D;
  __shared__ __align__(16) double stage[kRowGroups][kRowLanes][NEN * BS + 1];  // +1: no bank conflicts
  __shared__ uint16_t s_list[kRowGroups][NEN * kRowMaxDeg];                     // node's slot list
  __shared__ uint16_t s_off[kRowGroups][kMaxNodeAdj + 1];                       // its slot offsets
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x % kRowLanes, g = threadIdx.x / kRowLanes;
  const int my_i = (lane % BS) / D, my_k = lane % D;  // diagonal entry of lanes < BS
  for (int64_t idx = (int64_t)blockIdx.x * kRowGroups + g; idx < A.n_nodes;
       idx += (int64_t)gridDim.x * kRowGroups) {
    // nodes in Morton order: the readers of each element context run close together in time
    const int64_t n = A.node_order ? A.node_order[idx] : idx;
    const int64_t i0 = A.inc_ptr[n];
    const int deg = (int)(A.inc_ptr[n + 1] - i0);
    const int64_t a0 = A.nadj_ptr[n];
    const int sn = (int)(A.nadj_ptr[n + 1] - a0);
    if (deg == 0) continue;
    const unsigned bcn = A.node_bc ? A.node_bc[n] : 0u;
    for (int q = lane; q < NEN * deg; q += kRowLanes) s_list[g][q] = A.slot_list[NEN * i0 + q];
    for (int q = lane; q <= sn; q += kRowLanes) s_off[g][q] = A.slot_off[a0 + n + q];
    int ds = 0;  // slot of the diagonal block (node n itself)
    for (int base = 0; base < sn; base += kRowLanes) {
      const unsigned hit = __ballot_sync(FULL, base + lane < sn && A.nadj[a0 + base + lane] == n);
      if (hit) { ds = base + __ffs(hit) - 1; break; }
    }
    const int64_t rp_lane = lane < D ? A.row_ptr[n * D + lane] : 0;
    const int64_t rp_my = __shfl_sync(FULL, rp_lane, my_i);
    const uint16_t *sl = s_list[g];
    const uint16_t *so = s_off[g];
    double dsum = 0.0;  // diagonal-block entry (lanes < BS), summed over all incident elements
    for (int l0 = 0; l0 < deg; l0 += kRowLanes) {
      const int l = l0 + lane;
      double diag[BS];
#pragma unroll
      for (int q = 0; q < BS; ++q) diag[q] = 0.0;
      if (l < deg) {
        const int32_t packed = A.inc[i0 + l];
        const int a = packed % NEN;
        CtxLite<D> cx;
        load_ctx<D>(A.ctx, packed / NEN, cx);
        double Ga[D], ga[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          Ga[j] = cx.G[0][j];
          ga[j] = cx.g[0][j];
        }
#pragma unroll
        for (int q = 1; q < NEN; ++q)
          if (a == q) {
#pragma unroll
            for (int j = 0; j < D; ++j) {
              Ga[j] = cx.G[q][j];
              ga[j] = cx.g[q][j];
            }
          }
#pragma unroll
        for (int b = 0; b < NEN; ++b) {
          double GG = 0.0;
#pragma unroll
          for (int j = 0; j < D; ++j) GG = fma(Ga[j], cx.G[b][j], GG);
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const double ak = cx.sc1 * ga[k], bk = cx.sc2 * cx.g[b][k];
#pragma unroll
            for (int i = 0; i < D; ++i) {
              double t = fma(ak, cx.g[b][i], bk * ga[i]);
              if (i == k) t = fma(cx.smu, GG, t);
              if (b == a) diag[i * D + k] = t;                      // K_aa: warp-reduced
              else stage[g][lane][b * BS + i * D + k] = t;          // K_ab: slot lists
            }
          }
        }
      }
      // diagonal block: butterfly sum over the lanes (fixed order, identical on all lanes)
#pragma unroll
      for (int q = 0; q < BS; ++q) {
        double v = diag[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (q == lane) dsum += v;
      }
      __syncwarp();
      // off-diagonal blocks: lane s owns slot s (all BS entries, in registers) and sums
      // its slot list in order; partial sums of earlier chunks live in the output itself
      const bool first = (l0 == 0), last = (l0 + kRowLanes >= deg);
      for (int s = lane; s < sn; s += kRowLanes) {
        if (s == ds) continue;
        double acc[BS];
#pragma unroll
        for (int q = 0; q < BS; ++q) acc[q] = 0.0;
        if (!first) {
#pragma unroll
          for (int q = 0; q < BS; ++q) {
            if constexpr (TR)  // partial sums of earlier chunks at the transposed slot
              acc[q] = A.vals[rp_row(A, A.nadj[a0 + s], q % D) + (int64_t)A.tslot[a0 + s] * D + q / D];
            else
              acc[q] = A.vals[rp_row(A, n, q / D) + (int64_t)s * D + q % D];
          }
        }
        for (int c = so[s]; c < so[s + 1]; ++c) {
          const int ent = sl[c];
          const int le = (ent >> 2) - l0;
          if (le < 0 || le >= kRowLanes) continue;
          const double *st = &stage[g][le][(ent & 3) * BS];
#pragma unroll
          for (int q = 0; q < BS; ++q) acc[q] += st[q];
        }
        const int32_t m = A.nadj[a0 + s];
        const unsigned bcm = (last && A.node_bc) ? A.node_bc[m] : 0u;
        if constexpr (TR) {  // K[m D + k, n D + i] = K[n D + i, m D + k]
          const int64_t ts = A.tslot[a0 + s];
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const int64_t base = rp_row(A, m, k) + ts * D;
#pragma unroll
            for (int i = 0; i < D; ++i) {
              double v = acc[i * D + k];
              if (last && ((bcm >> k) & 1u)) v = 0.0;   // identity row of (m, k) (off-diagonal)
              if (last && ((bcn >> i) & 1u)) v = 0.0;   // masked column (n, i)
              A.vals[base + i] = v;
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < D; ++i) {
            const int64_t base = rp_row(A, n, i) + (int64_t)s * D;
#pragma unroll
            for (int k = 0; k < D; ++k) {
              double v = acc[i * D + k];
              if (last && ((bcm >> k) & 1u)) v = 0.0;     // masked column
              if (last && ((bcn >> i) & 1u)) v = 0.0;     // identity row (off-diagonal)
              A.vals[base + k] = v;
            }
          }
        }
      }
      __syncwarp();
    }
    if (lane < BS) {  // diagonal block
      double v = dsum;
      if (bcn & (1u << my_k)) v = 0.0;                                    // masked column
      if (bcn & (1u << my_i)) v = (my_k == my_i) ? 1.0 : 0.0;             // identity row
      A.vals[rp_my + (int64_t)ds * D + my_k] = v;
    }
    if (A.dmpc_ptr && lane < D) {  // B^T entries of row (n, lane), ascending constraint id
      const int64_t r = n * D + lane;
      const bool drow = bcn & (1u << lane);
      const int32_t lo = A.dmpc_ptr[r], hi = A.dmpc_ptr[r + 1];
      int64_t w = A.row_ptr[r] + (int64_t)sn * D;
      int32_t prev = -1;
      for (int32_t q = lo; q < hi; ++q, ++w) {
        int32_t kmin = INT32_MAX;
        for (int32_t q2 = lo; q2 < hi; ++q2) {
          const int32_t kk = A.dmpc[q2];
          if (kk > prev && kk < kmin) kmin = kk;
        }
        prev = kmin;
        const double v = (A.ms[kmin] == r ? 1.0 : 0.0) - (A.mm[kmin] == r ? 1.0 : 0.0);
        A.vals[w] = drow ? 0.0 : v;
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

// ------------------------------------------------------------------ element scatter-add (f1)
// The paper's comparison path (Fig. 4 right): one thread per
// element evaluates the dense element Hessian K^e (its (D+1)^2 blocks K_ab, the same
// closed form as the colored columns) and scatter-adds every entry into the CSR values with
// fp64 atomics — the "unstructured memory access ... atomic contention" the paper measures
// against.  The CSR position of block (a, b) row i column k is row_ptr[n_a D + i] +
// D * slot(n_b in the sorted neighbour list of n_a) + k (multiplier columns, if any, come
// after all u columns of a row).  Masked entries (Dirichlet row or column) are skipped;
// the unit diagonal of constrained DOFs and the Lagrangian blocks are written afterwards.
template <int D, int MAT>
__global__ void __launch_bounds__(kThreads) k_scatter_hessian(AsmArgs A, const int64_t *row_ptr,
                                                             const int64_t *nadj_ptr,
                                                             const int32_t *nadj, double *vals) {
  constexpr int NEN = D + 1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < A.E; e += stride) {
    int32_t nd[NEN];
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
    unsigned bc[NEN];
#pragma unroll
    for (int a = 0; a < NEN; ++a) bc[a] = A.node_bc ? __ldg(A.node_bc + nd[a]) : 0u;
#pragma unroll
    for (int a = 0; a < NEN; ++a) {
      const int64_t a0 = __ldg(nadj_ptr + nd[a]);
      const int sn = (int)(__ldg(nadj_ptr + nd[a] + 1) - a0);
      int64_t rows[D];
#pragma unroll
      for (int i = 0; i < D; ++i) rows[i] = __ldg(row_ptr + (int64_t)nd[a] * D + i);
#pragma unroll
      for (int b = 0; b < NEN; ++b) {
        int lo = 0, hi = sn;  // slot of nd[b] among nd[a]'s neighbours
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (__ldg(nadj + a0 + mid) < nd[b]) lo = mid + 1; else hi = mid;
        }
#pragma unroll
        for (int k = 0; k < D; ++k) {
          if (bc[b] & (1u << k)) continue;  // masked column
          double col[D];
          column_block<D>(cx, a, b, k, col);
#pragma unroll
          for (int i = 0; i < D; ++i) {
            if (bc[a] & (1u << i)) continue;  // masked row
            atomicAdd(vals + rows[i] + (int64_t)lo * D + k, col[i]);
          }
        }
      }
    }
  }
}

// B^T columns of the Lagrangian in the u rows: row s_k / m_k, column N_u + k = +1 / -1
// (0 when the row DOF is Dirichlet), found by binary search in the row.
__global__ void k_scatter_mpc_cols(const int32_t *ms, const int32_t *mm, int64_t nc, int64_t nu,
                                   int dim, const uint8_t *node_bc, const int64_t *row_ptr,
                                   const int32_t *col_idx, double *vals) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nc;
       k += (int64_t)gridDim.x * blockDim.x) {
    for (int side = 0; side < 2; ++side) {
      const int32_t r = side == 0 ? ms[k] : mm[k];
      const bool d = node_bc && (node_bc[r / dim] & (1u << (r % dim)));
      int64_t lo = row_ptr[r], hi = row_ptr[r + 1];
      const int32_t c = (int32_t)(nu + k);
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (col_idx[mid] < c) lo = mid + 1; else hi = mid;
      }
      vals[lo] = d ? 0.0 : (side == 0 ? 1.0 : -1.0);
    }
  }
}

__global__ void k_unit_diag(const int32_t *dofs, int64_t nd, const int64_t *diag_pos, double *vals) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nd;
       q += (int64_t)gridDim.x * blockDim.x)
    vals[diag_pos[dofs[q]]] = 1.0;
}

fem_status morton_node_order(Problem *p, cudaStream_t s);

static fem_status build_slot_lists(Problem *p, cudaStream_t s) {
  if (p->slot_list || p->n_nodes == 0) return FEM_OK;
  const int64_t nent = p->n_elems * p->nen * p->nen;
  const int64_t nnode_nnz = p->n_nodes + (p->n_nodes > 0 ? 0 : 0);
  int64_t nadj_total = 0;
  FEM_CUDA(cudaMemcpyAsync(&nadj_total, p->nadj_ptr + p->n_nodes, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  FEM_CUDA(cudaMalloc(&p->slot_list, sizeof(uint16_t) * (nent > 0 ? nent : 1)));
  FEM_CUDA(cudaMalloc(&p->slot_off, sizeof(uint16_t) * (nadj_total + nnode_nnz + 1)));
  if (p->dim == 2)
    k_slot_build<2><<<grid_for(p->n_nodes, 128), 128, 0, s>>>(p->inc_ptr, p->inc, p->conn, p->nadj_ptr, p->nadj, p->n_nodes, p->slot_list, p->slot_off, p->d_err);
  else
    k_slot_build<3><<<grid_for(p->n_nodes, 128), 128, 0, s>>>(p->inc_ptr, p->inc, p->conn, p->nadj_ptr, p->nadj, p->n_nodes, p->slot_list, p->slot_off, p->d_err);
  FEM_LAUNCH_CHECK("slot lists");
  fem_status st = morton_node_order(p, s);
  if (st) return st;
  return read_error_word(p, s);
}

template <int D, int MAT>
static void launch_colored(const AsmArgs &a, bool literal, int pass, cudaStream_t s) {
  const int grid = grid_for(a.E);
  if (literal) k_colored_hvp<D, MAT, true><<<grid, kThreads, 0, s>>>(a, pass);
  else k_colored_hvp<D, MAT, false><<<grid, kThreads, 0, s>>>(a, pass);
}

// tslot[nadj_ptr[n] + s] = index of n in the (sorted) adjacency of its s-th neighbour
__global__ void k_transpose_slots(const int64_t *nadj_ptr, const int32_t *nadj, int64_t n_nodes,
                                  uint8_t *tslot) {
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x)
    for (int64_t q = nadj_ptr[n]; q < nadj_ptr[n + 1]; ++q) {
      const int32_t m = nadj[q];
      int64_t lo = nadj_ptr[m], hi = nadj_ptr[m + 1];
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) / 2;
        if (nadj[mid] <= n) lo = mid;
        else hi = mid;
      }
      tslot[q] = (uint8_t)(lo - nadj_ptr[m]);
    }
}

// FEM_ASSEMBLE_COLORED: setup (node colors from the DOF coloring, color = colors[n D] / D;
// seed lists per color in Morton order; transposed slots; slot lists) and one launch of
// k_rows_fused<D, true> per node color.
static fem_status assemble_colored(Problem *p, const double *z, double *vals, bool bc,
                                   cudaStream_t s) {
  if (p->n_mpc) {
    set_error("FEM_ASSEMBLE_COLORED: multipliers not supported (use the default row form)");
    return FEM_ERR_INVALID_ARG;
  }
  fem_status st = build_slot_lists(p, s);   // also the Morton node order
  if (st) return st;
  const int D = p->dim;
  if (!p->ncolor_list) {
    std::vector<int32_t> col((size_t)p->N), order((size_t)p->n_nodes);
    FEM_CUDA(cudaMemcpyAsync(col.data(), p->colors, sizeof(int32_t) * p->N, cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaMemcpyAsync(order.data(), p->node_order, sizeof(int32_t) * p->n_nodes, cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaStreamSynchronize(s));
    const int ncol = (p->n_colors + D - 1) / D;
    std::vector<int64_t> cnt(ncol + 1, 0);
    for (int64_t n = 0; n < p->n_nodes; ++n) ++cnt[col[n * D] / D + 1];
    p->ncolor_off.assign(ncol + 1, 0);
    for (int c = 0; c < ncol; ++c) p->ncolor_off[c + 1] = p->ncolor_off[c] + cnt[c + 1];
    std::vector<int64_t> fill(p->ncolor_off.begin(), p->ncolor_off.end() - 1);
    std::vector<int32_t> list((size_t)p->n_nodes);
    for (int64_t q = 0; q < p->n_nodes; ++q) {
      const int32_t n = order[q];
      list[fill[col[(int64_t)n * D] / D]++] = n;
    }
    FEM_CUDA(cudaMalloc(&p->ncolor_list, sizeof(int32_t) * (p->n_nodes > 0 ? p->n_nodes : 1)));
    FEM_CUDA(cudaMemcpyAsync(p->ncolor_list, list.data(), sizeof(int32_t) * p->n_nodes, cudaMemcpyHostToDevice, s));
    int64_t nadj_total = 0;
    FEM_CUDA(cudaMemcpyAsync(&nadj_total, p->nadj_ptr + p->n_nodes, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaStreamSynchronize(s));
    FEM_CUDA(cudaMalloc(&p->tslot, nadj_total > 0 ? nadj_total : 1));
    k_transpose_slots<<<grid_for(p->n_nodes), kThreads, 0, s>>>(p->nadj_ptr, p->nadj, p->n_nodes, p->tslot);
    FEM_LAUNCH_CHECK("transposed slots");
  }
  // node tiles of one color each (contexts in shared memory, transposed stores); the warp
  // pull over HBM context records below is the fallback for meshes the tile plan rejects
  st = build_colored_tiles(p, s);
  if (st) return st;
  if (p->ct.state == 1 && !getenv("FEM_COLORED_PULL")) return launch_colored_tiles(p, z, vals, bc, s);
  RowArgs A{};
  A.node_bc = bc ? p->node_bc : nullptr; A.z = z;
  A.inc_ptr = p->inc_ptr; A.inc = p->inc; A.nadj_ptr = p->nadj_ptr; A.nadj = p->nadj;
  A.slot_list = p->slot_list; A.slot_off = p->slot_off;
  A.row_ptr = p->row_ptr; A.n_u = p->n_u; A.vals = vals; A.err = p->d_err; A.dim = D;
  A.tslot = p->tslot;
  const int st_ctx = D == 3 ? ctx_stride<3>() : ctx_stride<2>();
  st = ensure(p->ctxbuf, sizeof(double) * (size_t)st_ctx * (p->n_elems > 0 ? p->n_elems : 1));
  if (st) return st;
  A.ctx = (const double *)p->ctxbuf.ptr;
  if (p->n_elems) {   // tangent contexts in caller element order (p->inc indexes them)
    const int ge = grid_for(p->n_elems, kCtxThreads);
    double *ctx = (double *)p->ctxbuf.ptr;
    if (D == 2) {
      if (p->material == FEM_LINEAR_ELASTIC) k_elem_ctx<2, FEM_LINEAR_ELASTIC><<<ge, kCtxThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, nullptr, ctx, p->d_err);
      else k_elem_ctx<2, FEM_NEO_HOOKEAN><<<ge, kCtxThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, nullptr, ctx, p->d_err);
    } else {
      if (p->material == FEM_LINEAR_ELASTIC) k_elem_ctx<3, FEM_LINEAR_ELASTIC><<<ge, kCtxThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, nullptr, ctx, p->d_err);
      else k_elem_ctx<3, FEM_NEO_HOOKEAN><<<ge, kCtxThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, nullptr, ctx, p->d_err);
    }
  }
  for (size_t c = 0; c + 1 < p->ncolor_off.size(); ++c) {
    A.node_order = p->ncolor_list + p->ncolor_off[c];
    A.n_nodes = p->ncolor_off[c + 1] - p->ncolor_off[c];
    if (A.n_nodes == 0) continue;
    const int grid = grid_for(A.n_nodes, kRowGroups, 148 * 64);
    if (D == 2) k_rows_fused<2, true><<<grid, kRowLanes * kRowGroups, 0, s>>>(A);
    else k_rows_fused<3, true><<<grid, kRowLanes * kRowGroups, 0, s>>>(A);
  }
  FEM_LAUNCH_CHECK("fused colored assembly");
  return FEM_OK;
}

static fem_status assemble(Problem *p, const double *z, double *vals, unsigned flags,
                           cudaStream_t s) {
  const bool bc = (flags & FEM_APPLY_BC) && p->n_dir;
  if (flags & FEM_ASSEMBLE_COLORED) return assemble_colored(p, z, vals, bc, s);
  if (flags & FEM_ASSEMBLE_SCATTER) {
    FEM_CUDA(cudaMemsetAsync(vals, 0, sizeof(double) * (size_t)p->nnz, s));
    AsmArgs a{};
    a.coords = p->coords; a.conn = p->conn; a.E = p->n_elems; a.lam = p->lam; a.mu = p->mu;
    a.phase = p->phase; a.lam_tab = p->lam_tab; a.mu_tab = p->mu_tab;
    a.node_bc = bc ? p->node_bc : nullptr; a.z = z; a.err = p->d_err;
    if (p->n_elems) {
      const int g = grid_for(p->n_elems);
      if (p->dim == 2) {
        if (p->material == FEM_LINEAR_ELASTIC) k_scatter_hessian<2, FEM_LINEAR_ELASTIC><<<g, kThreads, 0, s>>>(a, p->row_ptr, p->nadj_ptr, p->nadj, vals);
        else k_scatter_hessian<2, FEM_NEO_HOOKEAN><<<g, kThreads, 0, s>>>(a, p->row_ptr, p->nadj_ptr, p->nadj, vals);
      } else {
        if (p->material == FEM_LINEAR_ELASTIC) k_scatter_hessian<3, FEM_LINEAR_ELASTIC><<<g, kThreads, 0, s>>>(a, p->row_ptr, p->nadj_ptr, p->nadj, vals);
        else k_scatter_hessian<3, FEM_NEO_HOOKEAN><<<g, kThreads, 0, s>>>(a, p->row_ptr, p->nadj_ptr, p->nadj, vals);
      }
    }
    if (p->n_mpc) {
      k_scatter_mpc_cols<<<grid_for(p->n_mpc), kThreads, 0, s>>>(p->mpc_s, p->mpc_m, p->n_mpc, p->n_u, p->dim, bc ? p->node_bc : nullptr, p->row_ptr, p->col_idx, vals);
      k_rows_mpc<<<grid_for(p->n_mpc), kThreads, 0, s>>>(p->mpc_s, p->mpc_m, p->n_mpc, p->n_u, p->dim, bc ? p->node_bc : nullptr, p->row_ptr, vals);
    }
    if (bc) k_unit_diag<<<grid_for(p->n_dir), kThreads, 0, s>>>(p->dir_dofs, p->n_dir, p->diag_pos, vals);
    FEM_LAUNCH_CHECK("scatter-add assembly");
    return FEM_OK;
  }
  // default: the row form (node tiles; fallbacks below); explicit mode flags override
  const bool rows = (flags & FEM_ASSEMBLE_ROWS) ||
                    !(flags & (FEM_ASSEMBLE_LITERAL | FEM_ASSEMBLE_JCOMP));
  if (rows) {
    fem_status st0 = build_row_tiles(p, s);
    if (st0) return st0;
    if (p->rt.state == 1) {
      st0 = launch_row_tiles(p, z, vals, bc, s);
      if (st0) return st0;
      if (p->n_mpc) {  // the Lagrangian's B^T columns in the u rows and the multiplier rows
        k_scatter_mpc_cols<<<grid_for(p->n_mpc), kThreads, 0, s>>>(p->mpc_s, p->mpc_m, p->n_mpc, p->n_u, p->dim, bc ? p->node_bc : nullptr, p->row_ptr, p->col_idx, vals);
        k_rows_mpc<<<grid_for(p->n_mpc), kThreads, 0, s>>>(p->mpc_s, p->mpc_m, p->n_mpc, p->n_u, p->dim, bc ? p->node_bc : nullptr, p->row_ptr, vals);
        FEM_LAUNCH_CHECK("row tiles: Lagrangian entries");
      }
      return FEM_OK;
    }
    st0 = build_row_plan(p, s);
    if (st0) return st0;
    if (p->rp_state != 1) {
      st0 = build_slot_lists(p, s);
      if (st0) return st0;
    }
    RowArgs A{};
    A.coords = p->coords; A.conn = p->conn; A.lam = p->lam; A.mu = p->mu;
    A.phase = p->phase; A.lam_tab = p->lam_tab; A.mu_tab = p->mu_tab;
    A.node_bc = bc ? p->node_bc : nullptr; A.z = z;
    A.inc_ptr = p->inc_ptr; A.inc = p->inc; A.nadj_ptr = p->nadj_ptr; A.nadj = p->nadj;
    A.slot_list = p->slot_list; A.slot_off = p->slot_off; A.node_order = p->node_order;
    A.dmpc_ptr = p->dmpc_ptr; A.dmpc = p->dmpc; A.ms = p->mpc_s; A.mm = p->mpc_m;
    A.row_ptr = p->row_ptr; A.n_nodes = p->n_nodes; A.n_u = p->n_u; A.vals = vals; A.err = p->d_err;
    A.dim = p->dim;
    // per-element tangent context, then the row-pull
    const int st_ctx = p->dim == 3 ? ctx_stride<3>() : ctx_stride<2>();
    fem_status stc = ensure(p->ctxbuf, sizeof(double) * (size_t)st_ctx * (p->n_elems > 0 ? p->n_elems : 1));
    if (stc) return stc;
    A.ctx = (const double *)p->ctxbuf.ptr;
    if (p->n_elems) {
      const int ge = grid_for(p->n_elems, kCtxThreads);
      double *ctx = (double *)p->ctxbuf.ptr;
      const int32_t *perm = p->rp_state == 1 ? p->tiles.perm : nullptr;
      if (p->dim == 2) {
        if (p->material == FEM_LINEAR_ELASTIC) k_elem_ctx<2, FEM_LINEAR_ELASTIC><<<ge, kCtxThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, perm, ctx, p->d_err);
        else k_elem_ctx<2, FEM_NEO_HOOKEAN><<<ge, kCtxThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, perm, ctx, p->d_err);
      } else {
        if (p->material == FEM_LINEAR_ELASTIC) k_elem_ctx<3, FEM_LINEAR_ELASTIC><<<ge, kCtxThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, perm, ctx, p->d_err);
        else k_elem_ctx<3, FEM_NEO_HOOKEAN><<<ge, kCtxThreads, 0, s>>>(p->coords, p->conn, p->n_elems, p->lam, p->mu, p->phase, p->lam_tab, p->mu_tab, z, perm, ctx, p->d_err);
      }
    }
    if (p->rp_state == 1)
      return launch_rows_pull(p, A.ctx, vals, bc, s);
    const int grid = grid_for(p->n_nodes, kRowGroups, 148 * 64);
    if (p->dim == 2) k_rows_fused<2><<<grid, kRowLanes * kRowGroups, 0, s>>>(A);
    else k_rows_fused<3><<<grid, kRowLanes * kRowGroups, 0, s>>>(A);
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
  k_decompress<<<grid_for(p->N * 8, kThreads, 148 * 32), kThreads, 0, s>>>(p->row_ptr, p->col_idx, p->colors, J, C, p->N, vals);
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

// Node-block SpMV for patterns of full D x D node blocks (no multiplier columns): the D rows
// of node n share one column list (the D * sn columns of its sn neighbour nodes, sorted), so
// the kernel reads the neighbour list nadj (4 B per block) instead of col_idx (4 B per
// entry), and each neighbour's D x-values once for the D rows.  LPN lanes per node, lane s =
// neighbour slot s; per row the lanes' partial sums are reduced by a butterfly.
template <int D, int LPN>
__global__ void __launch_bounds__(256) k_spmv_nodes(const int64_t *row_ptr, const int64_t *nadj_ptr,
                                                    const int32_t *nadj, const double *vals,
                                                    const double *x, double *y, int64_t n_nodes) {
  const int lane = threadIdx.x % LPN;
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x / LPN);
  for (int64_t n = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPN; n < n_nodes; n += groups) {
    const int64_t a0 = __ldg(nadj_ptr + n);
    const int sn = (int)(__ldg(nadj_ptr + n + 1) - a0);
    const int64_t rp0 = __ldg(row_ptr + n * D);
    double acc[D];
#pragma unroll
    for (int i = 0; i < D; ++i) acc[i] = 0.0;
    for (int sl = lane; sl < sn; sl += LPN) {
      const int64_t m = __ldg(nadj + a0 + sl);
      double xm[D];
#pragma unroll
      for (int k = 0; k < D; ++k) xm[k] = __ldg(x + m * D + k);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const double *v = vals + rp0 + (int64_t)i * D * sn + sl * D;
#pragma unroll
        for (int k = 0; k < D; ++k) acc[i] = fma(__ldg(v + k), xm[k], acc[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int o = LPN / 2; o > 0; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o, LPN);
    if (lane < D) {
      double v = acc[0];
#pragma unroll
      for (int i = 1; i < D; ++i)
        if (lane == i) v = acc[i];
      y[n * D + lane] = v;
    }
  }
}

__global__ void k_max_adj(const int64_t *nadj_ptr, int64_t n, int *mx) {
  int m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (int)(nadj_ptr[i + 1] - nadj_ptr[i]));
  atomicMax(mx, m);
}

fem_status run_spmv(Problem *p, const double *vals, const double *x, double *y, cudaStream_t s) {
  if (p->spmv_lpn == 0) {  // node-block form available? (pattern of full node blocks)
    p->spmv_lpn = -1;
    if (p->n_mpc == 0 && p->n_nodes > 0 && !getenv("FEM_SPMV_CSR")) {
      int *d = nullptr, h = 0;
      FEM_CUDA(cudaMalloc(&d, sizeof(int)));
      FEM_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s));
      k_max_adj<<<grid_for(p->n_nodes), kThreads, 0, s>>>(p->nadj_ptr, p->n_nodes, d);
      FEM_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s));
      FEM_CUDA(cudaStreamSynchronize(s));
      cudaFree(d);
      p->spmv_lpn = h <= 8 ? 8 : (h <= 16 ? 16 : 32);
    }
  }
  if (p->spmv_lpn > 0) {
    const int lpn = p->spmv_lpn;
    const int grid = grid_for(p->n_nodes * lpn, 256, 148 * 32);
    if (p->dim == 3) {
      if (lpn == 8) k_spmv_nodes<3, 8><<<grid, 256, 0, s>>>(p->row_ptr, p->nadj_ptr, p->nadj, vals, x, y, p->n_nodes);
      else if (lpn == 16) k_spmv_nodes<3, 16><<<grid, 256, 0, s>>>(p->row_ptr, p->nadj_ptr, p->nadj, vals, x, y, p->n_nodes);
      else k_spmv_nodes<3, 32><<<grid, 256, 0, s>>>(p->row_ptr, p->nadj_ptr, p->nadj, vals, x, y, p->n_nodes);
    } else {
      if (lpn == 8) k_spmv_nodes<2, 8><<<grid, 256, 0, s>>>(p->row_ptr, p->nadj_ptr, p->nadj, vals, x, y, p->n_nodes);
      else if (lpn == 16) k_spmv_nodes<2, 16><<<grid, 256, 0, s>>>(p->row_ptr, p->nadj_ptr, p->nadj, vals, x, y, p->n_nodes);
      else k_spmv_nodes<2, 32><<<grid, 256, 0, s>>>(p->row_ptr, p->nadj_ptr, p->nadj, vals, x, y, p->n_nodes);
    }
  } else {
    const int64_t avg = p->N ? p->nnz / p->N : 0;
    const int64_t threads_needed = p->N * (avg > 24 ? 8 : 4);
    const int grid = grid_for(threads_needed, 256, 148 * 32);
    if (avg > 24) k_spmv<8><<<grid, 256, 0, s>>>(p->row_ptr, p->col_idx, vals, x, y, p->N);
    else k_spmv<4><<<grid, 256, 0, s>>>(p->row_ptr, p->col_idx, vals, x, y, p->N);
  }
  FEM_LAUNCH_CHECK("spmv");
  if (p->size > 1) return halo_add(p, y, s);
  return FEM_OK;
}

fem_status run_assemble(Problem *p, const double *z, double *vals, unsigned flags, cudaStream_t s) {
  // Alg. 2 needs the coloring; the scatter-add comparison path only the pattern
  fem_status st = (flags & FEM_ASSEMBLE_SCATTER) ? build_pattern(p, s) : build_colors(p, s);
  if (st) return st;
  return assemble(p, z, vals, flags, s);
}

}  // namespace fem

using namespace fem;

extern "C" {

fem_status fem_assemble_csr(fem_problem *h, const double *z, double *vals, unsigned flags,
                            fem_stream stream) {
  FEM_NVTX_RANGE("fem_assemble_csr");
  FEM_ARG(h && z && vals, "fem_assemble_csr: null argument");
  return run_assemble(&h->p, z, vals, flags, (cudaStream_t)stream);
}

fem_status fem_spmv(fem_problem *h, const double *vals, const double *x, double *y,
                    fem_stream stream) {
  FEM_NVTX_RANGE("fem_spmv");
  FEM_ARG(h && vals && x && y, "fem_spmv: null argument");
  FEM_ARG(h->p.have_pattern, "fem_spmv: call fem_sparsity first");
  FEM_ARG(x != y, "fem_spmv: x and y alias");
  return run_spmv(&h->p, vals, x, y, (cudaStream_t)stream);
}

}  // extern "C"
