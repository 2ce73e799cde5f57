// fem_rows.cu — staged row-pull assembly of the sparse tangent (the FEM_ASSEMBLE_ROWS form
// of Alg. 2, reading R3): every CSR row block K_nm = sum_{e ∋ n,m} K^e_{a(n) b(m)}
// evaluated from the per-element context records of k_elem_ctx (fem_assemble.cu) and
// written once, no atomics, fixed summation order.
//
// One warp per node n, nodes in Morton order, persistent grid.  Per node:
//   1. TMA bulk copies bring the records of n's deg incident elements (one cp.async.bulk of
//      176 bytes each) and n's block list (setup-time plan, below) into shared memory,
//      completing on a per-buffer mbarrier; they are issued one node ahead, so the copies
//      of node k+1 overlap the arithmetic of node k;
//   2. lane l = incidence l completes (G_0, g_0) = -sum_b (G_b, g_b) in its record;
//   3. lane s = CSR slot s walks its run of the block list — the entries (l, a, b) of the
//      elements containing edge (n, nadj[s]), ascending element order — and accumulates
//      K^e_ab[i][k] = smu (G_a.G_b) d_ik + sc1 g_a[k] g_b[i] + sc2 g_a[i] g_b[k] from the
//      two record parts; lanes 28..31 walk a quarter each of the diagonal run (l, a, a),
//      and lanes 0..D*D-1 add the four partials in fixed order.
// Eligible meshes (build_row_plan): no MPC multiplier columns, <= 32 incidences and <= 28
// neighbours per node; otherwise the assembly falls back to k_rows_fused (fem_assemble.cu).
#include <cuda_runtime.h>

#include <cstdlib>

#include "fem_internal.cuh"

namespace fem {

#ifndef FEM_ROWS2_MINB
#define FEM_ROWS2_MINB 4
#endif
constexpr int kStageWarps = 4;
constexpr int kDiagLane0 = 28;  // lanes 28..31 walk the diagonal run

template <int D>
struct StageGeom {
  static constexpr int NEN = D + 1, BS = D * D, CS = ctx_stride<D>(), NP = 2 * D;
  static constexpr int RS0 = NP + CS;                                // (G_0 g_0) + record
  static constexpr int RS = ((RS0 / 2) % 2 == 0) ? RS0 + 2 : RS0;   // odd # of 16-byte units
  static constexpr int SC = NEN * NP;                                // smu, sc1, sc2
};

__host__ __device__ constexpr int entry_stride(int is, int nen) { return (nen * is + 7) & ~7; }

// ------------------------------------------------------------------ setup: the plan
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

// One thread per plan position idx (node n = node_order[idx]): incidences, the block list
// grouped by CSR slot (slot of a block = position of node b in n's sorted neighbour list),
// the slot offsets, the Dirichlet bits of the slot nodes, and the row start of n.
template <int D>
__global__ void k_plan_build(const int32_t *node_order, const int64_t *inc_ptr,
                             const int32_t *inc, const int32_t *conn, const int64_t *nadj_ptr,
                             const int32_t *nadj, const int64_t *row_ptr, const uint8_t *node_bc,
                             int64_t n_nodes, int IS, int ES, int SS, int4 *rp_node,
                             int32_t *rp_inc, uint16_t *rp_ent, uint8_t *rp_soff, uint8_t *rp_sbc,
                             int *bad) {
  constexpr int NEN = D + 1;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n_nodes;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int32_t n = node_order[idx];
    const int64_t i0 = inc_ptr[n], a0 = nadj_ptr[n];
    const int deg = (int)(inc_ptr[n + 1] - i0), sn = (int)(nadj_ptr[n + 1] - a0);
    if (deg > IS || sn + 1 > SS || deg > 32 || sn > kDiagLane0) { atomicOr(bad, 1); continue; }
    auto slot_of = [&](int32_t m) {
      int lo = 0, hi = sn;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (nadj[a0 + mid] < m) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    const int ds = sn > 0 ? slot_of(n) : 0;
    const int64_t rp0 = row_ptr[(int64_t)n * D];
    for (int i = 1; i <= D; ++i)  // rows of n: exactly D*sn columns each (no multiplier columns)
      if (row_ptr[(int64_t)n * D + i] != rp0 + (int64_t)i * D * sn) atomicOr(bad, 1);
    uint8_t cur[kDiagLane0 + 2];
    for (int q = 0; q <= sn; ++q) cur[q] = 0;
    for (int l = 0; l < deg; ++l) {
      const int32_t pk = inc[i0 + l];
      const int64_t e = pk / NEN;
      const int a = pk % NEN;
      for (int t = 0; t < NEN - 1; ++t) cur[slot_of(conn[e * NEN + (a + 1 + t) % NEN]) + 1]++;
    }
    for (int q = 0; q < sn; ++q) cur[q + 1] += cur[q];
    for (int q = 0; q <= sn; ++q) rp_soff[idx * SS + q] = cur[q];
    for (int q = 0; q < sn; ++q) rp_sbc[idx * SS + q] = node_bc ? node_bc[nadj[a0 + q]] : 0;
    uint16_t *ent = rp_ent + idx * ES;
    for (int q = 0; q < ES; ++q) ent[q] = 0;
    for (int l = 0; l < IS; ++l) {
      int32_t pk = -1;
      if (l < deg) {
        pk = inc[i0 + l];
        const int64_t e = pk / NEN;
        const int a = pk % NEN;
        for (int t = 0; t < NEN - 1; ++t) {
          const int b = (a + 1 + t) % NEN;
          ent[cur[slot_of(conn[e * NEN + b])]++] = (uint16_t)(l | a << 5 | b << 7);
        }
        ent[(NEN - 1) * deg + l] = (uint16_t)(l | a << 5 | a << 7);  // diagonal run
      }
      rp_inc[idx * IS + l] = pk;
    }
    const unsigned bcn = node_bc ? node_bc[n] : 0u;
    rp_node[idx] = make_int4(n, deg | sn << 8 | ds << 16 | (int)(bcn << 24),
                             (int)(uint32_t)(rp0 & 0xffffffffu), (int)(rp0 >> 32));
  }
}

fem_status build_row_plan(Problem *p, cudaStream_t s) {
  if (p->rp_state) return FEM_OK;
  p->rp_state = -1;
  if (p->n_mpc || p->n_nodes == 0 || p->n_elems == 0 || getenv("FEM_ROWS_LEGACY")) return FEM_OK;
  int *d_w = nullptr;
  FEM_CUDA(cudaMalloc(&d_w, 3 * sizeof(int)));
  FEM_CUDA(cudaMemsetAsync(d_w, 0, 3 * sizeof(int), s));
  k_plan_max<<<grid_for(p->n_nodes), kThreads, 0, s>>>(p->inc_ptr, p->nadj_ptr, p->n_nodes, d_w);
  int h_w[3] = {0, 0, 0};
  FEM_CUDA(cudaMemcpyAsync(h_w, d_w, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  if (h_w[0] > 32 || h_w[1] > kDiagLane0 || h_w[0] == 0) {
    cudaFree(d_w);
    return FEM_OK;
  }
  fem_status st = morton_node_order(p, s);
  if (st) { cudaFree(d_w); return st; }
  const int IS = h_w[0], ES = entry_stride(IS, p->nen), SS = (h_w[1] + 1 + 3) & ~3;
  const int64_t n = p->n_nodes;
  // +32 slack: every lane of a warp may load its word of the plan unconditionally
  FEM_CUDA(cudaMalloc(&p->rp_node, sizeof(int4) * n));
  FEM_CUDA(cudaMalloc(&p->rp_inc, sizeof(int32_t) * (n * IS + 32)));
  FEM_CUDA(cudaMalloc(&p->rp_ent, sizeof(uint16_t) * n * ES));
  FEM_CUDA(cudaMalloc(&p->rp_soff, (size_t)n * SS + 32));
  FEM_CUDA(cudaMalloc(&p->rp_sbc, (size_t)n * SS + 32));
  FEM_CUDA(cudaMemsetAsync(p->rp_inc + n * IS, 0xff, sizeof(int32_t) * 32, s));
  FEM_CUDA(cudaMemsetAsync(p->rp_soff + n * SS, 0, 32, s));
  FEM_CUDA(cudaMemsetAsync(p->rp_sbc + n * SS, 0, 32, s));
  if (p->dim == 2)
    k_plan_build<2><<<grid_for(n, 128), 128, 0, s>>>(p->node_order, p->inc_ptr, p->inc, p->conn, p->nadj_ptr, p->nadj, p->row_ptr, p->node_bc, n, IS, ES, SS, p->rp_node, p->rp_inc, p->rp_ent, p->rp_soff, p->rp_sbc, d_w + 2);
  else
    k_plan_build<3><<<grid_for(n, 128), 128, 0, s>>>(p->node_order, p->inc_ptr, p->inc, p->conn, p->nadj_ptr, p->nadj, p->row_ptr, p->node_bc, n, IS, ES, SS, p->rp_node, p->rp_inc, p->rp_ent, p->rp_soff, p->rp_sbc, d_w + 2);
  FEM_LAUNCH_CHECK("row plan");
  FEM_CUDA(cudaMemcpyAsync(h_w + 2, d_w + 2, sizeof(int), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  cudaFree(d_w);
  if (h_w[2]) {
    void *b[] = {p->rp_node, p->rp_inc, p->rp_ent, p->rp_soff, p->rp_sbc};
    for (void *x : b) cudaFree(x);
    p->rp_node = nullptr; p->rp_inc = nullptr; p->rp_ent = nullptr; p->rp_soff = nullptr; p->rp_sbc = nullptr;
    return FEM_OK;
  }
  p->rp_is = IS;
  p->rp_es = ES;
  p->rp_ss = SS;
  p->rp_state = 1;
  return FEM_OK;
}

// ------------------------------------------------------------------ async-copy primitives
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *m, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(m)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *m) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(m))
      : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// ------------------------------------------------------------------ kernel
struct StageArgs {
  const double *ctx;
  const int4 *node;
  const int32_t *inc;
  const uint16_t *ent;
  const uint8_t *soff, *sbc;
  int64_t n_nodes;
  int IS, ES, SS, bc;
  double *vals;
};

// (G_b, g_b) of a record part (16-byte aligned: 2*D doubles)
template <int D>
__device__ __forceinline__ void load_part(const double *rp, double (&G)[D], double (&g)[D]) {
  double v[2 * D];
#pragma unroll
  for (int j = 0; j < 2 * D; j += 2) {
    const double2 u = *reinterpret_cast<const double2 *>(rp + j);
    v[j] = u.x;
    v[j + 1] = u.y;
  }
#pragma unroll
  for (int j = 0; j < D; ++j) {
    G[j] = v[j];
    g[j] = v[D + j];
  }
}

// the block K^e_ab of list entry (l, a, b), added to acc
template <int D>
struct Contrib {
  double Ga[D], ga[D], Gb[D], gb[D], smu, sc1, sc2;
  __device__ __forceinline__ void load(const double *recs, uint32_t en) {
    using Gm = StageGeom<D>;
    const double *r = recs + (en & 31u) * Gm::RS;
    load_part<D>(r + ((en >> 5) & 3u) * Gm::NP, Ga, ga);
    load_part<D>(r + ((en >> 7) & 3u) * Gm::NP, Gb, gb);
    const double2 s01 = *reinterpret_cast<const double2 *>(r + Gm::SC);
    smu = s01.x;
    sc1 = s01.y;
    sc2 = r[Gm::SC + 2];
  }
  __device__ __forceinline__ void add_to(double (&acc)[D * D]) const {
    double dd = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) dd = fma(Ga[j], Gb[j], dd);
    dd *= smu;
    double p[D], q[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      p[j] = sc1 * ga[j];
      q[j] = sc2 * ga[j];
    }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int k = 0; k < D; ++k) {
        double v = fma(p[k], gb[i], q[i] * gb[k]);
        if (i == k) v += dd;
        acc[i * D + k] += v;
      }
  }
};

template <int D>
__global__ void __launch_bounds__(32 * kStageWarps, FEM_ROWS2_MINB) k_rows_stage(StageArgs A) {
  using Gm = StageGeom<D>;
  constexpr int NEN = Gm::NEN, BS = Gm::BS, NP = Gm::NP, RS = Gm::RS, CS = Gm::CS;
  extern __shared__ __align__(16) double sm_stage[];
  __shared__ __align__(8) uint64_t mbar[kStageWarps][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * kStageWarps;
  const int REC = A.IS * RS;                         // doubles of records per buffer
  const int BUF = REC + A.ES / 4;                    // + the block list (ES uint16)
  double *const bufs = sm_stage + (size_t)w * 2 * BUF;
  if (lane == 0) {
    mbar_init(&mbar[w][0], 1);
    mbar_init(&mbar[w][1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const int64_t last = A.n_nodes - 1;
  // plan words of position idx (clamped: loads are unconditional, validity is idx <= last)
  auto meta = [&](int64_t idx, int4 &nd, int32_t &pi) {
    const int64_t j = idx < last ? idx : last;
    nd = __ldg(A.node + j);
    pi = __ldg(A.inc + j * A.IS + lane);
  };
  auto issue = [&](int64_t idx, const int4 &nd, int32_t pi, int b) {
    double *dst = bufs + b * BUF;
    const int deg = nd.y & 0xff;
    if (lane == 0) {
      mbar_arrive_tx(&mbar[w][b], (unsigned)(deg * CS * sizeof(double) + A.ES * sizeof(uint16_t)));
      bulk_g2s(dst + REC, A.ent + idx * A.ES, A.ES * sizeof(uint16_t), &mbar[w][b]);
    }
    __syncwarp();
    if (lane < deg)
      bulk_g2s(dst + lane * RS + NP, A.ctx + (int64_t)(pi / NEN) * CS, CS * sizeof(double),
               &mbar[w][b]);
  };
  int64_t idx = (int64_t)blockIdx.x * kStageWarps + w;
  int4 nd_c, nd_n, nd_nn;
  int32_t pi_c, pi_n, pi_nn;
  meta(idx, nd_c, pi_c);
  if (idx <= last) issue(idx, nd_c, pi_c, 0);
  meta(idx + nw, nd_n, pi_n);
  for (int it = 0; idx <= last; ++it, idx += nw) {
    const int b = it & 1;
    double *cur = bufs + b * BUF;
    if (idx + nw <= last) issue(idx + nw, nd_n, pi_n, b ^ 1);  // in flight during this node
    meta(idx + 2 * nw, nd_nn, pi_nn);
    const int deg = nd_c.y & 0xff, sn = (nd_c.y >> 8) & 0xff, ds = (nd_c.y >> 16) & 0xff;
    const unsigned bcn = A.bc ? ((unsigned)nd_c.y >> 24) : 0u;
    const int64_t rp0 = (int64_t)(uint32_t)nd_c.z | ((int64_t)nd_c.w << 32);
    // this lane's run of the block list: CSR slot `lane`, or a quarter of the diagonal run
    int lo = __ldg(A.soff + idx * A.SS + lane), hi = __ldg(A.soff + idx * A.SS + lane + 1);
    const unsigned sbc = A.bc ? __ldg(A.sbc + idx * A.SS + lane) : 0u;
    const bool slot_lane = lane < sn && lane != ds;
    if (lane >= kDiagLane0) {
      const int j = lane - kDiagLane0;
      lo = (NEN - 1) * deg + (j * deg) / 4;
      hi = (NEN - 1) * deg + ((j + 1) * deg) / 4;
    } else if (!slot_lane) {
      lo = hi = 0;
    }
    mbar_wait(&mbar[w][b], (unsigned)(it >> 1) & 1u);
    if (lane < deg) {  // (G_0, g_0) = -sum of the other parts, in place
      double *r = cur + lane * RS;
#pragma unroll
      for (int j = 0; j < NP; j += 2) {
        double2 t = make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 1; q < NEN; ++q) {
          const double2 u = *reinterpret_cast<const double2 *>(r + q * NP + j);
          t.x += u.x;
          t.y += u.y;
        }
        *reinterpret_cast<double2 *>(r + j) = make_double2(-t.x, -t.y);
      }
    }
    __syncwarp();
    const uint16_t *ent = reinterpret_cast<const uint16_t *>(cur + REC);
    double acc[BS];
#pragma unroll
    for (int q = 0; q < BS; ++q) acc[q] = 0.0;
    int c = lo;
    for (; c + 1 < hi; c += 2) {
      Contrib<D> u, v;
      u.load(cur, ent[c]);
      v.load(cur, ent[c + 1]);
      u.add_to(acc);
      v.add_to(acc);
    }
    if (c < hi) {
      Contrib<D> u;
      u.load(cur, ent[c]);
      u.add_to(acc);
    }
    if (slot_lane) {
      double *row = A.vals + rp0 + lane * D;
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
    __syncwarp();  // records consumed: lanes 28..31 park their diagonal partials
    if (lane >= kDiagLane0) {
      double *st = cur + (lane - kDiagLane0) * BS;
#pragma unroll
      for (int q = 0; q < BS; ++q) st[q] = acc[q];
    }
    __syncwarp();
    if (lane < BS && deg > 0) {
      const int i = lane / D, k = lane % D;
      double v = cur[lane];
#pragma unroll
      for (int j = 1; j < 4; ++j) v += cur[j * BS + lane];
      if (bcn & (1u << k)) v = 0.0;                         // masked column
      if (bcn & (1u << i)) v = (i == k) ? 1.0 : 0.0;        // identity row
      A.vals[rp0 + (int64_t)i * D * sn + ds * D + k] = v;
    }
    fence_async_smem();  // generic accesses to this buffer precede the next bulk copy into it
    __syncwarp();
    nd_c = nd_n; pi_c = pi_n;
    nd_n = nd_nn; pi_n = pi_nn;
  }
}

template <int D>
static fem_status launch_stage(Problem *p, const double *ctx, double *vals, bool bc,
                               cudaStream_t s) {
  StageArgs A{};
  A.ctx = ctx; A.node = p->rp_node; A.inc = p->rp_inc; A.ent = p->rp_ent;
  A.soff = p->rp_soff; A.sbc = p->rp_sbc; A.n_nodes = p->n_nodes; A.IS = p->rp_is;
  A.ES = p->rp_es; A.SS = p->rp_ss; A.bc = bc ? 1 : 0; A.vals = vals;
  const size_t buf = sizeof(double) * (size_t)p->rp_is * StageGeom<D>::RS + sizeof(uint16_t) * p->rp_es;
  const size_t smem = (size_t)kStageWarps * 2 * buf;
  FEM_CUDA(cudaFuncSetAttribute(k_rows_stage<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  FEM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rows_stage<D>, 32 * kStageWarps, smem));
  int dev = 0, sms = 148;
  FEM_CUDA(cudaGetDevice(&dev));
  FEM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  const int64_t need = (p->n_nodes + kStageWarps - 1) / kStageWarps;
  if (grid > need) grid = need;
  k_rows_stage<D><<<(int)grid, 32 * kStageWarps, smem, s>>>(A);
  FEM_LAUNCH_CHECK("staged row assembly");
  return FEM_OK;
}

fem_status launch_rows_stage(Problem *p, const double *ctx, double *vals, bool bc,
                             cudaStream_t s) {
  return p->dim == 2 ? launch_stage<2>(p, ctx, vals, bc, s) : launch_stage<3>(p, ctx, vals, bc, s);
}

}  // namespace fem
