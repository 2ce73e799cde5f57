// fem_rows.cu — row-pull assembly of the sparse tangent (the FEM_ASSEMBLE_ROWS form of
// Alg. 2, reading R3): every CSR row block K_nm = sum_{e ∋ n,m} K^e_{a(n) b(m)}
// evaluated from the per-element context records of k_elem_ctx (fem_assemble.cu) and
// written once, no atomics, fixed summation order.
//
// Element blocks: with spatial gradients g = F^{-T} G and the record scalars smu = vol mu,
// sc1 = vol (mu - lambda ln J), sc2 = vol lambda,
//   K^e_ab[i][k] = smu (G_a.G_b) d_ik + sc1 g_a[k] g_b[i] + sc2 g_a[i] g_b[k].
// Since sum_b G_b = sum_b g_b = 0, every element row sums to zero over b (the energy is
// translation invariant), so the diagonal block of a row is minus the sum of its
// off-diagonal blocks: K_nn = -sum_{m != n} K_nm.  Only the off-diagonal blocks are summed
// from element entries (3 per incidence in 3D instead of 4).
//
// Work decomposition: nodes in Morton order (records in the element tiles' Morton order),
// LPN lanes per node (16: two consecutive nodes per warp), lane q = off-diagonal CSR slot q
// of its node.  The lane walks its run of the node's block list — the elements containing
// edge (n, nadj[s]), ascending element order, each entry (record, a, b) — loading the two
// record parts and the scalars straight from L1/L2 (the records of neighbouring nodes
// overlap, no shared-memory staging, so occupancy is set by registers), and writes its
// D x D block; the node's lanes then write the diagonal block (-sum of the slots, fixed
// order) with the Dirichlet mask.
// Eligible meshes (build_row_plan): no MPC multiplier columns, <= 32 off-diagonal slots per
// node, < 2^27 elements; otherwise the assembly falls back to k_rows_fused.
#include <cuda_runtime.h>

#include <cstdlib>
#include <vector>

#include "fem_internal.cuh"

namespace fem {

#ifndef FEM_ROWS_WARPS
#define FEM_ROWS_WARPS 8
#endif
#ifndef FEM_ROWS_MINB
#define FEM_ROWS_MINB 3
#endif
constexpr int kRowWarps = FEM_ROWS_WARPS;
constexpr uint32_t kPosBits = 27;

template <int D>
struct RecGeom {
  static constexpr int NEN = D + 1, BS = D * D, CS = ctx_stride<D>(), NP = 2 * D;
  static constexpr int SC = NEN * NP;                                // smu, sc1, sc2
  static constexpr int BP = (BS + 1) & ~1;                           // scratch block pitch
};

// ------------------------------------------------------------------ setup: the plan
__global__ void k_inverse_perm(const int32_t *perm, int64_t n, int32_t *pos) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    pos[perm[i]] = (int32_t)i;
}

__global__ void k_plan_max(const int64_t *inc_ptr, const int64_t *nadj_ptr, int64_t n, int *mx) {
  int d = 0, s = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    d = max(d, (int)(inc_ptr[i + 1] - inc_ptr[i]));
    s = max(s, (int)(nadj_ptr[i + 1] - nadj_ptr[i]));
  }
  atomicMax(mx, d);
  atomicMax(mx + 1, s);
}

// One thread per node position idx: the node word, the off-diagonal block list grouped by
// CSR slot (entries pos | a << 27 | b << 29, pos = record position of the element, ascending
// element order within a slot), the slot offsets and the Dirichlet bits of the slot nodes.
template <int D>
__global__ void k_plan_nodes(const int32_t *node_order, const int64_t *inc_ptr,
                             const int32_t *inc, const int32_t *conn, const int32_t *epos,
                             const int64_t *nadj_ptr, const int32_t *nadj, const int64_t *row_ptr,
                             const uint8_t *node_bc, int64_t n_nodes, int ES, int SS,
                             int4 *rp_node, uint32_t *rp_ent, uint8_t *rp_soff, uint8_t *rp_sbc,
                             int *bad) {
  constexpr int NEN = D + 1;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n_nodes;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int32_t n = node_order[idx];
    const int64_t i0 = inc_ptr[n], a0 = nadj_ptr[n];
    const int deg = (int)(inc_ptr[n + 1] - i0), sn = (int)(nadj_ptr[n + 1] - a0);
    auto slot_of = [&](int32_t mm) {
      int lo = 0, hi = sn;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (nadj[a0 + mid] < mm) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    const int ds = sn > 0 ? slot_of(n) : 0;
    const int sno = sn > 0 ? sn - 1 : 0;  // off-diagonal slots
    if (sn == 0 || ds >= sn || nadj[a0 + ds] != n || sno > 32 || (NEN - 1) * deg > ES ||
        (NEN - 1) * deg > 255) {
      atomicOr(bad, 1);
      continue;
    }
    const int64_t rp0 = row_ptr[(int64_t)n * D];
    for (int i = 1; i <= D; ++i)  // rows of n: exactly D*sn columns each (no multiplier columns)
      if (row_ptr[(int64_t)n * D + i] != rp0 + (int64_t)i * D * sn) atomicOr(bad, 1);
    uint8_t cnt[34];
    for (int q = 0; q <= sno; ++q) cnt[q] = 0;
    auto q_of = [&](int s) { return s < ds ? s : s - 1; };  // off-diagonal slot index
    for (int l = 0; l < deg; ++l) {
      const int32_t pk = inc[i0 + l];
      const int64_t e = pk / NEN;
      const int a = pk % NEN;
      for (int t = 1; t < NEN; ++t) cnt[q_of(slot_of(conn[e * NEN + (a + t) % NEN])) + 1]++;
    }
    for (int q = 0; q < sno; ++q) cnt[q + 1] += cnt[q];
    for (int q = 0; q <= sno; ++q) rp_soff[idx * SS + q] = cnt[q];
    for (int q = 0; q < sno; ++q) rp_sbc[idx * SS + q] = node_bc ? node_bc[nadj[a0 + q + (q >= ds)]] : 0;
    uint32_t *ent = rp_ent + idx * ES;
    for (int l = 0; l < deg; ++l) {
      const int32_t pk = inc[i0 + l];
      const int64_t e = pk / NEN;
      const int a = pk % NEN;
      const uint32_t pos = (uint32_t)epos[e];
      for (int t = 1; t < NEN; ++t) {
        const int b = (a + t) % NEN;
        ent[cnt[q_of(slot_of(conn[e * NEN + b]))]++] = pos | (uint32_t)a << kPosBits | (uint32_t)b << (kPosBits + 2);
      }
    }
    const unsigned bcn = node_bc ? node_bc[n] : 0u;
    rp_node[idx] = make_int4(n, sno | sn << 8 | ds << 16 | (int)(bcn << 24),
                             (int)(uint32_t)(rp0 & 0xffffffffu), (int)(rp0 >> 32));
  }
}

fem_status build_row_plan(Problem *p, cudaStream_t s) {
  if (p->rp_state) return FEM_OK;
  p->rp_state = -1;
  if (p->n_mpc || p->n_nodes == 0 || p->n_elems == 0 || p->n_elems >= (int64_t(1) << kPosBits) ||
      getenv("FEM_ROWS_LEGACY"))
    return FEM_OK;
  int *d_w = nullptr;
  FEM_CUDA(cudaMalloc(&d_w, 4 * sizeof(int)));
  FEM_CUDA(cudaMemsetAsync(d_w, 0, 4 * sizeof(int), s));
  k_plan_max<<<grid_for(p->n_nodes), kThreads, 0, s>>>(p->inc_ptr, p->nadj_ptr, p->n_nodes, d_w);
  int h_w[4] = {0, 0, 0, 0};
  FEM_CUDA(cudaMemcpyAsync(h_w, d_w, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  const int IS = h_w[0], max_sn = h_w[1];
  if (IS == 0 || max_sn - 1 > 32 || (p->nen - 1) * IS > 255) { cudaFree(d_w); return FEM_OK; }
  fem_status st = morton_node_order(p, s);
  if (!st) st = build_tiles(p, s);  // records are written in the element tiles' Morton order
  if (st) { cudaFree(d_w); return st; }
  const int64_t n = p->n_nodes, E = p->n_elems;
  const int lpn = (max_sn - 1 <= 16) ? 16 : 32;
  const int npw = 32 / lpn;
  const int ES = ((p->nen - 1) * IS + 3) & ~3, SS = (lpn + 1 + 3) & ~3;
  const int64_t npad = (n + npw - 1) / npw * npw;
  FEM_CUDA(cudaMalloc(&p->epos, sizeof(int32_t) * E));
  k_inverse_perm<<<grid_for(E), kThreads, 0, s>>>(p->tiles.perm, E, p->epos);
  FEM_CUDA(cudaMalloc(&p->rp_node, sizeof(int4) * npad));
  FEM_CUDA(cudaMalloc(&p->rp_ent, sizeof(uint32_t) * npad * ES));
  FEM_CUDA(cudaMalloc(&p->rp_soff, (size_t)npad * SS));
  FEM_CUDA(cudaMalloc(&p->rp_sbc, (size_t)npad * SS));
  FEM_CUDA(cudaMemsetAsync(p->rp_node, 0, sizeof(int4) * npad, s));
  FEM_CUDA(cudaMemsetAsync(p->rp_soff, 0, (size_t)npad * SS, s));
  FEM_CUDA(cudaMemsetAsync(p->rp_sbc, 0, (size_t)npad * SS, s));
  if (p->dim == 2)
    k_plan_nodes<2><<<grid_for(n, 128), 128, 0, s>>>(p->node_order, p->inc_ptr, p->inc, p->conn, p->epos, p->nadj_ptr, p->nadj, p->row_ptr, p->node_bc, n, ES, SS, p->rp_node, p->rp_ent, p->rp_soff, p->rp_sbc, d_w + 2);
  else
    k_plan_nodes<3><<<grid_for(n, 128), 128, 0, s>>>(p->node_order, p->inc_ptr, p->inc, p->conn, p->epos, p->nadj_ptr, p->nadj, p->row_ptr, p->node_bc, n, ES, SS, p->rp_node, p->rp_ent, p->rp_soff, p->rp_sbc, d_w + 2);
  FEM_LAUNCH_CHECK("row plan (nodes)");
  FEM_CUDA(cudaMemcpyAsync(h_w + 2, d_w + 2, sizeof(int), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_w);
  if (h_w[2]) {
    void *b[] = {p->epos, p->rp_node, p->rp_ent, p->rp_soff, p->rp_sbc};
    for (void *x : b) if (x) cudaFree(x);
    p->epos = nullptr; p->rp_node = nullptr; p->rp_ent = nullptr; p->rp_soff = nullptr;
    p->rp_sbc = nullptr;
    return FEM_OK;
  }
  p->rp_lpn = lpn;
  p->rp_es = ES;
  p->rp_ss = SS;
  p->rp_state = 1;
  return FEM_OK;
}

// ------------------------------------------------------------------ kernel
struct RowPullArgs {
  const double *ctx;
  const int4 *node;
  const uint32_t *ent;
  const uint8_t *soff, *sbc;
  int64_t n_nodes, n_units;
  int ES, SS, bc;
  double *vals;
};

template <int D>
__device__ __forceinline__ void ldg_part(const double *rp, double (&G)[D], double (&g)[D]) {
  double v[2 * D];
#pragma unroll
  for (int j = 0; j < 2 * D; j += 2) {
    const double2 u = __ldg(reinterpret_cast<const double2 *>(rp + j));
    v[j] = u.x;
    v[j + 1] = u.y;
  }
#pragma unroll
  for (int j = 0; j < D; ++j) {
    G[j] = v[j];
    g[j] = v[D + j];
  }
}

// LPN lanes per node (16: two consecutive nodes per warp), lane q = off-diagonal slot q:
// the lane loads the entries of its run (up to KE up front), sums their element blocks
// straight from the records and writes its D x D block; the node's lanes then write the
// diagonal block = -sum of the slots (ascending slot order) with the Dirichlet mask.
// (A/B, profiles/: entry-parallel lanes with shared-memory staged blocks 8.9 ms, row
// stores through shared memory 7.3 ms, cp.async-staged chunk records 8.4 ms, TMA per
// record 5.1 ms, this form 5.2 ms + 1.3 ms records at cfg 3.)
template <int D, int LPN>
__global__ void __launch_bounds__(32 * kRowWarps, FEM_ROWS_MINB) k_rows_pull(RowPullArgs A) {
  using Gm = RecGeom<D>;
  constexpr int BS = Gm::BS, NP = Gm::NP, CS = Gm::CS, BP = Gm::BP;
  constexpr int NPW = 32 / LPN;
  constexpr uint32_t PMASK = (1u << kPosBits) - 1u;
  __shared__ __align__(16) double scratch[kRowWarps][32 * BP];  // slot sums (diagonal)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int h = lane / LPN, ql = lane % LPN;
  double *scr = scratch[w];
  const int64_t W = (int64_t)gridDim.x * kRowWarps;
  constexpr int KE = 8;  // entries per lane loaded up front (longer runs loop)
  // node words of unit u (the plan arrays are padded: loads need no bounds)
  struct Unit { int4 nd; int lo, hi; unsigned sbc; };
  auto fetch = [&](int64_t u) {
    Unit x{make_int4(0, 0, 0, 0), 0, 0, 0u};
    if (u < A.n_units) {
      const int64_t idx = u * NPW + h;
      x.nd = __ldg(A.node + idx);
      x.lo = __ldg(A.soff + idx * A.SS + ql);
      x.hi = __ldg(A.soff + idx * A.SS + ql + 1);
      x.sbc = A.bc ? __ldg(A.sbc + idx * A.SS + ql) : 0u;
    }
    return x;
  };
  int64_t u = (int64_t)blockIdx.x * kRowWarps + w;
  Unit cur = fetch(u);
  for (; u < A.n_units; u += W) {
    const Unit nx = fetch(u + W);  // in flight during this unit
    const int64_t idx = u * NPW + h;
    const int4 nd = cur.nd;
    const int sno = nd.y & 0xff;
    const int lo = ql < sno ? cur.lo : 0, hi = ql < sno ? cur.hi : 0;
    const uint32_t *ent = A.ent + idx * A.ES;
    uint32_t ens[KE];
#pragma unroll
    for (int t = 0; t < KE; ++t) ens[t] = (lo + t < hi) ? __ldg(ent + lo + t) : 0u;
    double acc[BS];
#pragma unroll
    for (int q = 0; q < BS; ++q) acc[q] = 0.0;
    auto add_entry = [&](uint32_t en) {
      const double *rr = A.ctx + (int64_t)(en & PMASK) * CS;
      double Ga[D], ga[D], Gb[D], gb[D];
      ldg_part<D>(rr + ((en >> kPosBits) & 3u) * NP, Ga, ga);
      ldg_part<D>(rr + ((en >> (kPosBits + 2)) & 3u) * NP, Gb, gb);
      const double2 s01 = __ldg(reinterpret_cast<const double2 *>(rr + Gm::SC));
      const double sc2 = __ldg(rr + Gm::SC + 2);
      double dd = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) dd = fma(Ga[j], Gb[j], dd);
      dd *= s01.x;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const double qi = sc2 * ga[i];
#pragma unroll
        for (int k = 0; k < D; ++k) {
          double v = fma(s01.y * ga[k], gb[i], acc[i * D + k]);
          v = fma(qi, gb[k], v);
          acc[i * D + k] = (i == k) ? v + dd : v;
        }
      }
    };
#pragma unroll
    for (int t = 0; t < KE; ++t)
      if (lo + t < hi) add_entry(ens[t]);
    for (int e = lo + KE; e < hi; ++e) add_entry(__ldg(ent + e));
    const int sn = (nd.y >> 8) & 0xff, ds = (nd.y >> 16) & 0xff;
    const unsigned bcn = A.bc ? ((unsigned)nd.y >> 24) : 0u;
    const int64_t rp0 = (int64_t)(uint32_t)nd.z | ((int64_t)nd.w << 32);
    const bool live = idx < A.n_nodes;
    if (live && ql < sno) {
      const unsigned sbc = cur.sbc;
      const int s = ql + (ql >= ds);
      double *row = A.vals + rp0 + s * D;
      if ((sbc | bcn) == 0u) {
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int k = 0; k < D; ++k) row[(int64_t)i * D * sn + k] = acc[i * D + k];
      } else {
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int k = 0; k < D; ++k) {
            double v = acc[i * D + k];
            if ((sbc >> k) & 1u) v = 0.0;  // masked column
            if ((bcn >> i) & 1u) v = 0.0;  // identity row (off-diagonal)
            row[(int64_t)i * D * sn + k] = v;
          }
      }
    }
    // diagonal block: -sum of the node's off-diagonal slots (unmasked), ascending slot order
#pragma unroll
    for (int q = 0; q < BS; ++q) scr[lane * BP + q] = acc[q];
    __syncwarp();
    if (live && ql < BS) {
      const int i = ql / D, k = ql % D;
      double v = 0.0;
      for (int t = 0; t < sno; ++t) v += scr[(h * LPN + t) * BP + ql];
      v = -v;
      if (bcn & (1u << k)) v = 0.0;                         // masked column
      if (bcn & (1u << i)) v = (i == k) ? 1.0 : 0.0;        // identity row
      A.vals[rp0 + (int64_t)i * D * sn + ds * D + k] = v;
    }
    __syncwarp();  // scratch is rewritten by the next iteration
    cur = nx;
  }
}

template <int D, int LPN>
static fem_status launch_pull(Problem *p, const double *ctx, double *vals, bool bc,
                              cudaStream_t s) {
  RowPullArgs A{};
  constexpr int NPW = 32 / LPN;
  A.ctx = ctx; A.node = p->rp_node; A.ent = p->rp_ent; A.soff = p->rp_soff; A.sbc = p->rp_sbc;
  A.n_nodes = p->n_nodes; A.n_units = (p->n_nodes + NPW - 1) / NPW;
  A.ES = p->rp_es; A.SS = p->rp_ss; A.bc = bc ? 1 : 0; A.vals = vals;
  auto kern = k_rows_pull<D, LPN>;
  int per_sm = 0;
  FEM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kRowWarps, 0));
  int dev = 0, sms = 148;
  FEM_CUDA(cudaGetDevice(&dev));
  FEM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int64_t need = (A.n_units + kRowWarps - 1) / kRowWarps;
  if (grid > need) grid = need;
  kern<<<(int)grid, 32 * kRowWarps, 0, s>>>(A);
  FEM_LAUNCH_CHECK("row-pull assembly");
  return FEM_OK;
}

fem_status launch_rows_pull(Problem *p, const double *ctx, double *vals, bool bc,
                             cudaStream_t s) {
  if (p->dim == 2)
    return p->rp_lpn == 16 ? launch_pull<2, 16>(p, ctx, vals, bc, s) : launch_pull<2, 32>(p, ctx, vals, bc, s);
  return p->rp_lpn == 16 ? launch_pull<3, 16>(p, ctx, vals, bc, s) : launch_pull<3, 32>(p, ctx, vals, bc, s);
}

}  // namespace fem
