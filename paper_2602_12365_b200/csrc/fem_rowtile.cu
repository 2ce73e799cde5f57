// fem_rowtile.cu — fused node-tile assembly of the sparse tangent (FEM_ASSEMBLE_ROWS form of
// Alg. 2, reading R3; default in 3D): no per-element records in HBM.
//
// Nodes in Morton order are cut into tiles of NT consecutive nodes, one tile per CTA
// iteration of a persistent grid.  Setup packs per tile one metadata block: the tile's
// element set (every element incident to a tile node), its halo nodes, the elements'
// halo-local connectivity, and per tile node its CSR row word, off-diagonal slot offsets,
// Dirichlet bits and block list (entries (element, a, b) grouped by CSR slot; by default
// co-scheduled so that the slot lanes of a node read the same element at the same step, see
// k_rt_plan).  Per tile the CTA
//   0. has the block and the halo nodes' coordinates and state copied into shared memory
//      by cp.async (metadata two tiles ahead, node data one tile ahead);
//   1. evaluates every tile element's tangent context once into shared memory: spatial
//      gradients g_a = F^{-T} G_a (a = 0..d), M_ab = vol mu G_a.G_b for the element's node
//      pairs, sc1 = vol (mu - lambda ln J), sc2 = vol lambda;
//   2. sums, with 16 lanes per tile node and lane q = off-diagonal slot q, the element blocks
//      K^e_ab[i][k] = M_ab d_ik + sc1 g_a[k] g_b[i] + sc2 g_a[i] g_b[k] of the slot's run and
//      writes the D x D block; the diagonal block is minus the sum of the row's off-diagonal
//      blocks (every element row sums to zero: sum_b G_b = sum_b g_b = 0), summed over the
//      node's slot lanes in ascending slot order through shared memory.
// Elements on tile boundaries are evaluated by each tile that touches them (~2x at NT = 32
// in 3D); in exchange the HBM traffic is the CSR values, the metadata and the node data —
// no context records.  Atomic-free, fixed order: bitwise reproducible.
// Eligible meshes: <= 16 off-diagonal slots per node, tile sets within the plan's capacity;
// otherwise the assembly falls back to the row-pull kernels.  MPC problems: the kernel writes
// the u-blocks of every row (each row's multiplier columns follow them) and the assembly
// adds the Lagrangian entries (B^T columns, multiplier rows) with two small kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "element.cuh"
#include "fem_internal.cuh"
#include "pipe.cuh"

#ifndef FEM_RT_DIAG_SMEM
#define FEM_RT_DIAG_SMEM 1
#endif
#ifndef FEM_RT_BPODD
#define FEM_RT_BPODD 1
#endif
#ifndef FEM_RT_UNROLL
#define FEM_RT_UNROLL 4
#endif
// diagnostics only (A/B timing of the two phases; results are wrong when set): 1 = skip the
// element contexts, 2 = skip the slot sums and stores
#ifndef FEM_RT_DIAG_SKIP
#define FEM_RT_DIAG_SKIP 0
#endif
#ifndef FEM_RT_MINB
#define FEM_RT_MINB 2
#endif
#ifndef FEM_RT_RSODD
#define FEM_RT_RSODD 1
#endif
#ifndef FEM_RT_RSPAD
#define FEM_RT_RSPAD 0
#endif
#ifndef FEM_RT_GPAD
#define FEM_RT_GPAD 0
#endif
#ifndef FEM_RT_NT
#define FEM_RT_NT 16
#endif
// tile metadata blocks by one TMA bulk copy per tile (mbarrier completion) instead of 16-byte
// cp.async per thread (the LDGSTS of the block took 38 M of the 711 M shared wavefronts per
// launch at cfg 3, 11.5 per instruction against 4 conflict-free)
#ifndef FEM_RT_TMA_META
#define FEM_RT_TMA_META 1
#endif
// bank-aware placement of the context records (16-lane tiles): a record's shared-memory
// bank class is its slot mod 16, so each element is given the class whose banks collide
// least with the elements the same node reads at the same co-scheduled step (greedy at setup,
// k_rt_plan); the half-warp of a node then reads its g_b / M_ab / g_a / sc words from spread
// banks (ncu r02: 4.8 wavefronts per slot-loop load against 2 conflict-free).  Measured (r02,
// cfg 3): the greedy lowers the modelled g_b wavefronts per half-warp step by 15 % only
// (FEM_RT_PLACE_DEBUG=1 prints the model: each element's four gradient banks are a rigid
// pattern shared by all its node-steps), ncu shows 4.74 vs 4.82 per load, and the padded
// record slots make the kernel slower (3.63 vs 3.54 ms) — off by default.  A micro-benchmark
// (tools/micro/lds64.cu) confirms the model: 64-bit loads are served per half-warp.
#ifndef FEM_CT_NT
#define FEM_CT_NT 4    // max seeds per colored node tile (FEM_ASSEMBLE_COLORED; A/B cfg 3: 2 / 4 / 6 / 8 / 16 -> 12.8 / 8.24 / 8.30 / 8.85 / 9.18 ms)
#endif
#ifndef FEM_RT_PLACE
#define FEM_RT_PLACE 0
#endif
// Bank-conflict-free context records (3D, 16 lanes per node, row form): the records are
// stored field-major (SoA) with a stride S = kRtSoaS = 4 (mod 16) words, so a 64-bit load
// of field w of record r hits bank pair (4 w + r) mod 16: records of different r mod 4 (the
// record's "color") never collide, g_b[i] of one record (field 3 b + i) covers four distinct
// bank pairs over b, and M_ab sits at field 11 + (a ^ b) + 4 [0 not in {a, b}] (the three
// pairs at a vertex have distinct a ^ b, i.e. K4's three perfect matchings).  The plan colors
// each tile's elements with 4 colors (balanced per tile node), places element k of color c at
// record 4 k + c, and co-schedules each node's slot runs so that the elements read at one step
// have distinct colors: every load of the slot sums is then one wavefront per half-warp
// (ncu r02: 4.8 wavefronts per warp-wide load against 2, LSU 73 % busy).  Idle steps are
// entry 0xffff (no load).  0 = the odd-stride record layout (FEM_RT_RSODD).
#ifndef FEM_RT_SOA
#define FEM_RT_SOA 0
#endif
// node staging: one thread per halo node (D copies each of x and z) instead of one per
// component (the i / D, i % D address math: ncu source counters r02, 172 M of the kernel's
// 1.79 G warp instructions in the staging loop)
// diagonal blocks: the sum over the node's slot lanes unrolled with predicated loads and two
// partial sums (even / odd slots) instead of a counted loop of dependent adds
#ifndef FEM_RT_DIAG_UNROLL
#define FEM_RT_DIAG_UNROLL 1
#endif
#ifndef FEM_RT_ISSUE_NODE
#define FEM_RT_ISSUE_NODE 1
#endif
// visit budget of the plan's depth-first co-schedule search per node and length (0: first fit)
#ifndef FEM_RT_SOA_DFS
#define FEM_RT_SOA_DFS 4000
#endif
// co-scheduled block lists (see k_rt_plan): 0 = each slot's run in ascending element order
#ifndef FEM_RT_SCHED
#define FEM_RT_SCHED 1
#endif
// element contexts in cofactor form with fem_rcp instead of geometry()'s IEEE divisions
#ifndef FEM_RT_COF
#define FEM_RT_COF 1
#endif

namespace fem {

constexpr int kRtNT = FEM_RT_NT;         // nodes per tile
constexpr int kRtUnroll = FEM_RT_UNROLL; // entries per unrolled step of the slot sums
constexpr int kRtThreads = 256;          // 8 warps, 2 nodes per warp per pass
// threads per CTA of the colored (TR) node tiles.  256-thread CTAs leave 3/4 of the lanes at the
// barrier with 4-seed tiles (ncu r02: 64 % barrier stalls), but smaller CTAs measured slower
// (cfg 3, colored Alg. 2: 64 threads 8.65 ms, 128 threads 9.05 / 8.85 ms with 4 / 8 seeds,
// 64 / 32 threads with 2 seeds 9.23 / 8.77 ms, against 8.28 ms at 256): 256 kept.
#ifndef FEM_CT_THREADS
#define FEM_CT_THREADS 256
#endif
#ifndef FEM_CT_MINB
#define FEM_CT_MINB 2
#endif
constexpr int rt_threads(bool tr) { return tr ? FEM_CT_THREADS : kRtThreads; }
constexpr int kRtLPNMax = 32;            // lanes per node: 8 (2D, <= 8 off-diagonal slots), 16 (3D Kuhn,
                                         // <= 16) or 32 (unstructured, 8-node tiles)
constexpr int kRtMaxSlots = 64;          // off-diagonal slots per node: a lane sums slots ql, ql + LPN, ...
constexpr int kRtSortMax = 4096;         // plan: keys sorted per tile in shared memory
constexpr int kRtSchedHist = 17;         // plan statistics: bad[1 + C] nodes with schedule length C, bad[1 + 17] grouped
constexpr int kRtSoaS = 324;             // SoA record stride (= 4 mod 16; records per tile <= 324)
constexpr int kRtSoaF = 20;              // SoA fields: g 0-11, M 12-14 / 16-18, sc1 15, sc2 19
static_assert(kRtSoaS % 16 == 4, "SoA stride must be 4 mod 16");
__host__ __device__ constexpr int rt_soa_m(int a, int b) { return 11 + (a ^ b) + ((a && b) ? 4 : 0); }

template <int D>
struct RtGeom {
  static constexpr int NEN = D + 1, BS = D * D, NPAIR = D == 3 ? 6 : 3;
  static constexpr int GP = FEM_RT_GPAD ? ((D + 1) & ~1) : D;     // g_a stride (padded: 16 B)
  static constexpr int G0 = 0, M0 = NEN * GP, S0 = M0 + NPAIR + (NPAIR & 1);  // g | M | sc1 sc2
  static constexpr int RS = (FEM_RT_RSODD ? ((S0 + 2) | 1) : (S0 + 2)) + FEM_RT_RSPAD;  // odd: spreads records over banks
  static constexpr int BP = FEM_RT_BPODD ? (BS | 1) : ((BS + 1) & ~1);  // scratch block pitch
};

// index of the unordered node pair {a, b}: 3D (01 02 03 12 13 23), 2D (01 02 12)
// (a != b): 3D a + b - [0 in {a, b}], 2D a + b - 1 — three integer ops per slot-loop entry
// instead of the min / max / select chain
template <int D>
__host__ __device__ constexpr int rt_pair(int a, int b) {
  return D == 3 ? a + b - (a * b == 0 ? 1 : 0) : a + b - 1;
}

struct RtLayout {
  int nt, lpn, uem, unm, es, ss, mb;
  int soa;  // 1: SoA records (FEM_RT_SOA), uem = kRtSoaS
  int off_halo, off_lc, off_ph, off_nd, off_so, off_sb, off_en;
  int off_tb, off_tsn;  // TR (colored Alg. 2): per (node, slot) transposed block base, neighbour row length
};

static inline int r16(int x) { return (x + 15) & ~15; }

static RtLayout rt_layout(int nt, int lpn, int uem, int unm, int es, int ss, bool phase,
                          bool tr = false, bool soa = false) {
  RtLayout L{};
  L.nt = nt; L.lpn = lpn; L.uem = uem; L.unm = unm; L.es = es; L.ss = ss; L.soa = soa ? 1 : 0;
  L.off_halo = 16;
  L.off_lc = r16(L.off_halo + 4 * unm);
  L.off_ph = r16(L.off_lc + 8 * uem);
  L.off_nd = r16(L.off_ph + (phase ? uem : 0));
  L.off_so = r16(L.off_nd + 16 * nt);
  L.off_sb = r16(L.off_so + 2 * nt * ss);   // slot offsets: uint16
  L.off_en = r16(L.off_sb + nt * ss);
  L.off_tb = r16(L.off_en + 2 * nt * es);
  L.off_tsn = L.off_tb + (tr ? 8 * nt * ss : 0);
  L.mb = r16(L.off_tsn + (tr ? nt * ss : 0));
  return L;
}

// ------------------------------------------------------------------ setup
__device__ void rt_bitonic(int32_t *key, int m, int tid, int nthr) {
  int P = 1;
  while (P < m) P <<= 1;
  for (int i = m + tid; i < P; i += nthr) key[i] = INT32_MAX;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < P; i += nthr) {
        const int ij = i ^ j;
        if (ij > i) {
          const bool up = (i & k) == 0;
          const int32_t x = key[i], y = key[ij];
          if ((x > y) == up) { key[i] = y; key[ij] = x; }
        }
      }
      __syncthreads();
    }
}

// sorted unique in place (one thread), returns the count
__device__ int rt_unique(int32_t *key, int m) {
  int u = 0;
  for (int i = 0; i < m; ++i)
    if (i == 0 || key[i] != key[i - 1]) key[u++] = key[i];
  return u;
}

__device__ int rt_find(const int32_t *key, int n, int32_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (key[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// One CTA per tile.  count mode (meta == null): Ue, Un per tile (and a fail flag when the
// sort capacity is exceeded); fill mode: the packed metadata block.
template <int D>
__global__ void __launch_bounds__(256) k_rt_plan(const int32_t *node_order, int64_t n_nodes,
                                                 const int64_t *inc_ptr, const int32_t *inc,
                                                 const int32_t *conn, const uint8_t *phase,
                                                 const int64_t *nadj_ptr, const int32_t *nadj,
                                                 const int64_t *row_ptr, const uint8_t *node_bc,
                                                 RtLayout L, int32_t *cnt, uint8_t *meta,
                                                 int *bad) {
  constexpr int NEN = D + 1;
  __shared__ int32_t elems[kRtSortMax];
  __shared__ int32_t halo[kRtSortMax];
  __shared__ int s_m, s_ue, s_un;
  const int64_t t = blockIdx.x;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int64_t n0 = t * L.nt;
  const int nn = (int)((n_nodes - n0) < L.nt ? (n_nodes - n0) : L.nt);
  if (tid == 0) s_m = 0;
  __syncthreads();
  // incident elements of the tile's nodes
  for (int j = 0; j < nn; ++j) {
    const int32_t n = node_order[n0 + j];
    const int64_t i0 = inc_ptr[n];
    const int deg = (int)(inc_ptr[n + 1] - i0);
    const int base = s_m;
    if (base + deg > kRtSortMax) {
      if (tid == 0) atomicOr(bad, 1);
      return;
    }
    for (int l = tid; l < deg; l += nthr) elems[base + l] = inc[i0 + l] / NEN;
    __syncthreads();
    if (tid == 0) s_m = base + deg;
    __syncthreads();
  }
  rt_bitonic(elems, s_m, tid, nthr);
  if (tid == 0) s_ue = rt_unique(elems, s_m);
  __syncthreads();
  const int ue = s_ue;
  if (ue * NEN > kRtSortMax) {
    if (tid == 0) atomicOr(bad, 1);
    return;
  }
  for (int q = tid; q < ue * NEN; q += nthr) halo[q] = conn[(int64_t)elems[q / NEN] * NEN + q % NEN];
  __syncthreads();
  rt_bitonic(halo, ue * NEN, tid, nthr);
  if (tid == 0) s_un = rt_unique(halo, ue * NEN);
  __syncthreads();
  const int un = s_un;
  // SoA records (FEM_RT_SOA): 4-coloring of the tile's elements, balanced per tile node;
  // element k of color c at record 4 k + c (s_soa[0]: record of each element, s_soa[1]:
  // element of each record or 0xffff, s_soa[2]: tile-node mask of each element)
  __shared__ uint16_t s_soa[3][1024];
  __shared__ int s_nslot;
  const bool soa = L.soa != 0;
  if (soa) {
    if (ue > 1024) {
      if (tid == 0) atomicOr(bad, 1);
      return;
    }
    for (int e = tid; e < ue; e += nthr) {
      unsigned mk = 0;
      for (int a = 0; a < NEN; ++a) {
        const int32_t nd = conn[(int64_t)elems[e] * NEN + a];
        for (int j = 0; j < nn; ++j)
          if (node_order[n0 + j] == nd) mk |= 1u << j;
      }
      s_soa[2][e] = (uint16_t)mk;
    }
    __syncthreads();
    if (tid == 0) {
      uint8_t cn[16][4];
      int csz[4] = {0, 0, 0, 0};
      for (int j = 0; j < 16; ++j)
        for (int c = 0; c < 4; ++c) cn[j][c] = 0;
      for (int e = 0; e < ue; ++e) {
        const unsigned mk = s_soa[2][e];
        int bc = 0, bmax = 1 << 30, bsum = 1 << 30, bsz = 1 << 30;
        for (int c = 0; c < 4; ++c) {
          int mx = 0, sm = 0;
          for (int j = 0; j < 16; ++j)
            if (mk >> j & 1u) { mx = max(mx, cn[j][c] + 1); sm += cn[j][c]; }
          if (mx < bmax || (mx == bmax && (sm < bsum || (sm == bsum && csz[c] < bsz)))) {
            bc = c; bmax = mx; bsum = sm; bsz = csz[c];
          }
        }
        for (int j = 0; j < 16; ++j)
          if (mk >> j & 1u) ++cn[j][bc];
        s_soa[0][e] = (uint16_t)(4 * csz[bc] + bc);
        ++csz[bc];
      }
      const int ns = 4 * max(max(csz[0], csz[1]), max(csz[2], csz[3]));
      s_nslot = ns;
      for (int q = 0; q < ns && q < 1024; ++q) s_soa[1][q] = 0xffff;
      for (int e = 0; e < ue; ++e)
        if (s_soa[0][e] < 1024) s_soa[1][s_soa[0][e]] = (uint16_t)e;
    }
    __syncthreads();
  }
  // bank-aware placement: records in 16 bank classes of ceil(ue / 16) slots each
  const bool place = !soa && FEM_RT_PLACE && FEM_RT_SCHED && L.lpn == 16;
  const int nslot = soa ? s_nslot : place ? (ue + 15) & ~15 : ue;
  auto rec_of = [&](int r) -> int { return soa ? (int)s_soa[0][r] : r; };  // sorted index -> record
  if (!meta) {
    if (tid == 0) { cnt[2 * t] = nslot; cnt[2 * t + 1] = un; }
    return;
  }
  __shared__ uint8_t s_best[64];   // co-schedule length per tile node (0: grouped runs)
  for (int j = tid; j < 64; j += nthr) s_best[j] = 0;
  uint8_t *blk = meta + t * (int64_t)L.mb;
  if (tid == 0) {
    int *h = reinterpret_cast<int *>(blk);
    h[0] = soa ? nslot : ue; h[1] = un; h[2] = nn; h[3] = 0;
  }
  int32_t *hid = reinterpret_cast<int32_t *>(blk + L.off_halo);
  for (int q = tid; q < L.unm; q += nthr) hid[q] = q < un ? halo[q] : 0;
  uint16_t *lc = reinterpret_cast<uint16_t *>(blk + L.off_lc);
  for (int q = tid; q < L.uem * 4; q += nthr) {
    int e = q / 4;
    const int a = q % 4;
    uint16_t v = 0;
    if (soa) {  // records in slot order; holes marked lc.x = 0xffff
      e = e < nslot ? (int)s_soa[1][e] : 0xffff;
      if (e == 0xffff) v = a == 0 ? 0xffff : 0;
    }
    if (e < ue && a < NEN) v = (uint16_t)rt_find(halo, un, conn[(int64_t)elems[e] * NEN + a]);
    lc[q] = v;
  }
  if (phase) {
    uint8_t *ph = blk + L.off_ph;
    for (int q = tid; q < L.uem; q += nthr) {
      const int e = soa ? (q < nslot ? (int)s_soa[1][q] : 0xffff) : q;
      ph[q] = e < ue ? phase[elems[e]] : 0;
    }
  }
  // per tile node: row word, off-diagonal slots, block list
  int4 *ndw = reinterpret_cast<int4 *>(blk + L.off_nd);
  uint16_t *so = reinterpret_cast<uint16_t *>(blk + L.off_so);
  uint8_t *sb = blk + L.off_sb;
  uint16_t *en = reinterpret_cast<uint16_t *>(blk + L.off_en);
  for (int j = tid; j < L.nt; j += nthr) {
    ndw[j] = make_int4(0, 0, 0, 0);
    for (int q = 0; q < L.ss; ++q) { so[j * L.ss + q] = 0; sb[j * L.ss + q] = 0; }
    if (j >= nn) continue;
    const int32_t n = node_order[n0 + j];
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
    const int sno = sn > 0 ? sn - 1 : 0;
    if (sn == 0 || ds >= sn || nadj[a0 + ds] != n || sno > kRtMaxSlots || sno + 1 > L.ss ||
        (NEN - 1) * deg > L.es) {
      atomicOr(bad, 1);
      continue;
    }
    // row i of node n = D * sn u-columns (the node blocks) followed by its multiplier columns
    // (MPC Lagrangian, indices >= N_u): start = rp0 + i D sn + ex_i, ex_i = multiplier columns
    // of the node's rows before i (packed in the node word; <= 0xffff)
    const int64_t rp0 = row_ptr[(int64_t)n * D];
    int ex[4] = {0, 0, 0, 0};
    for (int i = 1; i <= D; ++i) {
      const int64_t extra = row_ptr[(int64_t)n * D + i] - (rp0 + (int64_t)i * D * sn);
      if (extra < 0 || extra > 0xffff || (i < D && extra > 0xffff)) atomicOr(bad, 1);
      ex[i] = (int)extra;
    }
    uint16_t c[kRtMaxSlots + 2];
    for (int q = 0; q <= sno; ++q) c[q] = 0;
    auto q_of = [&](int s) { return s < ds ? s : s - 1; };
    for (int l = 0; l < deg; ++l) {
      const int32_t pk = inc[i0 + l];
      const int64_t e = pk / NEN;
      const int a = pk % NEN;
      for (int k = 1; k < NEN; ++k) c[q_of(slot_of(conn[e * NEN + (a + k) % NEN])) + 1]++;
    }
    for (int q = 0; q < sno; ++q) c[q + 1] += c[q];
    for (int q = 0; q <= sno; ++q) so[j * L.ss + q] = c[q];
    for (int q = 0; q < sno; ++q) sb[j * L.ss + q] = node_bc ? node_bc[nadj[a0 + q + (q >= ds)]] : 0;
    if (L.off_tsn > L.off_tb) {  // TR: where K[m, n] (the transpose of slot q's block) lives
      int64_t *tb = reinterpret_cast<int64_t *>(blk + L.off_tb);
      uint8_t *tsn = blk + L.off_tsn;
      for (int q = 0; q < sno; ++q) {
        const int32_t mm = nadj[a0 + q + (q >= ds)];
        const int64_t b0 = nadj_ptr[mm];
        const int snm = (int)(nadj_ptr[mm + 1] - b0);
        int lo = 0, hi = snm;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (nadj[b0 + mid] < n) lo = mid + 1; else hi = mid;
        }
        tb[j * L.ss + q] = row_ptr[(int64_t)mm * D] + (int64_t)lo * D;  // row (m, 0), column block n
        tsn[j * L.ss + q] = (uint8_t)snm;
      }
    }
    uint16_t *ej = en + j * L.es;
    for (int q = 0; q < L.es; ++q) ej[q] = 0;
    const unsigned bcn = node_bc ? node_bc[n] : 0u;
    const int4 word = make_int4(ex[1] | (D == 3 ? ex[2] << 16 : 0),
                                sno | sn << 8 | ds << 16 | (int)(bcn << 24),
                                (int)(uint32_t)(rp0 & 0xffffffffu), (int)(rp0 >> 32));
#if FEM_RT_SCHED
    // Co-scheduling: the slot lanes of a node step through their runs in lock step; an element
    // incident to the node feeds 3 (2D: 2) slots.  Place each element at one iteration k of
    // all its slots' runs (first fit over a few deterministic element orders, the shortest
    // schedule kept), so the lanes reading that element's g_a, sc1, sc2 at step k read the
    // same shared-memory words (broadcast) instead of NEN-1 random records.  Idle steps point
    // at the zero record (index uem): exact no-op contributions.  Run q = entries
    // [q C, (q + 1) C).  Nodes whose schedule does not fit keep the grouped runs below.
    constexpr int kSchedMaxDeg = 64, kSchedMaxC = 15;
    int maxrun = 0;
    for (int q = 0; q < sno; ++q) maxrun = max(maxrun, (int)(c[q + 1] - c[q]));
    if (deg <= kSchedMaxDeg && maxrun > 0) {
      uint64_t msk[kSchedMaxDeg];
      uint8_t col[kSchedMaxDeg];   // SoA: record color (elements of one step: distinct colors)
      int ncol[4] = {0, 0, 0, 0};
      for (int l = 0; l < deg; ++l) {
        const int32_t pk = inc[i0 + l];
        const int64_t e = pk / NEN;
        const int a = pk % NEN;
        uint64_t mm = 0;
        for (int k = 1; k < NEN; ++k) mm |= 1ull << q_of(slot_of(conn[e * NEN + (a + k) % NEN]));
        msk[l] = mm;
        col[l] = soa ? (uint8_t)(rec_of(rt_find(elems, ue, (int32_t)e)) & 3) : 0;
        ++ncol[col[l]];
      }
      // lower bound of the schedule length: the longest run; SoA: also the largest color class
      const int lb = soa ? max(maxrun, max(max(ncol[0], ncol[1]), max(ncol[2], ncol[3]))) : maxrun;
      uint8_t perm[kSchedMaxDeg], it[kSchedMaxDeg];
      auto attempt = [&](int seed) -> int {  // returns the schedule length (kSchedMaxC + 1: failed)
        for (int l = 0; l < deg; ++l) perm[l] = (uint8_t)l;
        uint32_t st = 0x9e3779b9u * (uint32_t)(seed + 1);
        if (seed)
          for (int l = deg - 1; l > 0; --l) {  // Fisher-Yates with a fixed LCG
            st = st * 1664525u + 1013904223u;
            const int k = (int)((st >> 8) % (uint32_t)(l + 1));
            const uint8_t tmp = perm[l]; perm[l] = perm[k]; perm[k] = tmp;
          }
        uint64_t busy[kSchedMaxC];
        uint8_t cbusy[kSchedMaxC];
        for (int k = 0; k < kSchedMaxC; ++k) { busy[k] = 0; cbusy[k] = 0; }
        int C = 0;
        for (int x = 0; x < deg; ++x) {
          const int l = perm[x];
          const uint8_t cm = soa ? (uint8_t)(1u << col[l]) : 0;
          int k = 0;
          while (k < kSchedMaxC && ((busy[k] & msk[l]) || (cbusy[k] & cm))) ++k;
          if (k == kSchedMaxC) return kSchedMaxC + 1;
          busy[k] |= msk[l];
          cbusy[k] |= cm;
          it[l] = (uint8_t)k;
          C = max(C, k + 1);
        }
        return C;
      };
      int best = kSchedMaxC + 1, bseed = 0;
      for (int seed = 0; seed < 64 && best > lb; ++seed) {
        const int C = attempt(seed);
        if (C < best) { best = C; bseed = seed; }
      }
      // SoA: the color constraint makes first fit leave ~1.5 steps on the table (Kuhn: 7.9
      // steps against a bound of 6); a bounded depth-first search for C = lb .. best - 1
      // (empty steps are interchangeable: only the first one is tried) usually finds 7
      bool dfs_ok = false;
      if (soa && FEM_RT_SOA_DFS && best > lb) {
        int8_t st[kSchedMaxDeg];
        uint64_t busy[kSchedMaxC];
        uint8_t cbusy[kSchedMaxC];
        for (int C = lb; C < best && C <= kSchedMaxC && !dfs_ok; ++C) {
          for (int k = 0; k < C; ++k) { busy[k] = 0; cbusy[k] = 0; }
          int i = 0, visits = 0;
          st[0] = -1;
          while (i >= 0 && i < deg && visits < FEM_RT_SOA_DFS) {
            ++visits;
            const uint8_t cm = (uint8_t)(1u << col[i]);
            int k = st[i];
            if (k >= 0) {  // undo the previous placement of item i
              busy[k] &= ~msk[i];
              cbusy[k] &= (uint8_t)~cm;
              if (busy[k] == 0) { st[i] = -1; --i; continue; }  // it was an empty step
            }
            for (++k; k < C; ++k)
              if (!(busy[k] & msk[i]) && !(cbusy[k] & cm)) break;
            if (k < C) {
              busy[k] |= msk[i];
              cbusy[k] |= cm;
              st[i] = (int8_t)k;
              if (++i < deg) st[i] = -1;
            } else {
              st[i] = -1;
              --i;
            }
          }
          if (i == deg) {
            dfs_ok = true;
            best = C;
            for (int l = 0; l < deg; ++l) it[l] = (uint8_t)st[l];
          }
        }
      }
      if (best <= kSchedMaxC && sno * best <= L.es) {
        if (!dfs_ok) attempt(bseed);
        // idle steps: the zero record (AoS) or 0xffff (SoA: predicated off, no load)
        const uint16_t zero = soa ? (uint16_t)0xffff : (uint16_t)(L.uem | 0 << 10 | 1 << 12);
        for (int q = 0; q < sno * best; ++q) ej[q] = zero;
        for (int l = 0; l < deg; ++l) {
          const int32_t pk = inc[i0 + l];
          const int64_t e = pk / NEN;
          const int a = pk % NEN;
          const int r = rec_of(rt_find(elems, ue, (int32_t)e));
          for (int k = 1; k < NEN; ++k) {
            const int b = (a + k) % NEN;
            ej[q_of(slot_of(conn[e * NEN + b])) * best + it[l]] = (uint16_t)(r | a << 10 | b << 12);
          }
        }
        for (int q = 0; q <= sno; ++q) so[j * L.ss + q] = (uint16_t)(q * best);
        if (j < 64) s_best[j] = (uint8_t)best;
        atomicAdd(bad + 1 + best, 1);  // schedule-length histogram (FEM_RT_SCHED_STATS)
        ndw[j] = word;
        continue;
      }
    }
#endif
    atomicAdd(bad + 1 + kRtSchedHist, 1);  // nodes on grouped runs (no co-schedule)
    for (int l = 0; l < deg; ++l) {
      const int32_t pk = inc[i0 + l];
      const int64_t e = pk / NEN;
      const int a = pk % NEN;
      const int r = rec_of(rt_find(elems, ue, (int32_t)e));
      for (int k = 1; k < NEN; ++k) {
        const int b = (a + k) % NEN;
        ej[c[q_of(slot_of(conn[e * NEN + b]))]++] = (uint16_t)(r | a << 10 | b << 12);
      }
    }
    ndw[j] = word;
  }
  if (!place) return;
  // ---- bank-aware record placement (one thread; the per-node schedules are complete)
  __syncthreads();
  constexpr int RS = RtGeom<D>::RS;
  uint32_t *occ = reinterpret_cast<uint32_t *>(halo);   // [ue][4] (j | k << 8 | a << 16)
  int32_t *info = elems;                                  // [ue] count | slot << 8
  // addresses per bank of each load type (g_b, M_ab, g_a, sc) at each (warp, step): a warp's
  // 64-bit loads serve its two nodes' 32 lanes together (ncu: 2 wavefronts conflict-free)
  __shared__ uint8_t mk[4][8][16][16];
  if (tid == 0) {
    for (int r = 0; r < ue; ++r) info[r] = 0;
    for (int c = 0; c < 4 * 8 * 16 * 16; ++c) (&mk[0][0][0][0])[c] = 0;
    for (int j = 0; j < nn && j < 16; ++j) {
      const int best = s_best[j];
      if (!best) continue;
      const int sno = ndw[j].y & 0xff;
      const uint16_t *ej = en + j * L.es;
      for (int c = 0; c < sno * best; ++c) {
        const int r = ej[c] & 1023;
        if (r >= ue) continue;                            // zero record (idle step)
        const int k = c % best, a = (ej[c] >> 10) & 3;
        const int n = info[r] & 0xff;
        bool seen = false;
        for (int o = 0; o < n; ++o) seen |= (int)(occ[r * 4 + o] & 0xff) == j;
        if (!seen && n < 4) {
          occ[r * 4 + n] = (uint32_t)j | (uint32_t)k << 8 | (uint32_t)a << 16;
          info[r] = n + 1;
        }
      }
    }
    // slot classes: bank(slot) = RS slot mod 16 (RS odd: a bijection of slot mod 16)
    int cls_cnt[16];
    for (int c = 0; c < 16; ++c) cls_cnt[c] = 0;
    const int cap = (ue + 15) / 16;
    int rs_inv = 1;
    for (int x = 1; x < 16; x += 2) if (((RS * x) & 15) == 1) rs_inv = x;
    for (int want = 4; want >= 0; --want)  // most-constrained elements first
      for (int r = 0; r < ue; ++r) {
        const int n = info[r] & 0xff;
        if (n != want) continue;
        int bestc = -1, bcost = 1 << 30;
        for (int sg = 0; sg < 16; ++sg) {
          if (cls_cnt[sg] >= cap) continue;
          int cost = 0;
          for (int o = 0; o < n; ++o) {
            const uint32_t w = occ[r * 4 + o];
            const int j = (w & 0xff) >> 1, k = (w >> 8) & 0xff, a = (w >> 16) & 3;
            for (int b = 0; b < NEN; ++b) {
              if (b == a) continue;
              cost += 3 * mk[0][j][k][(sg + 3 * b) & 15];
              cost += mk[1][j][k][(sg + RtGeom<D>::M0 + rt_pair<D>(a, b)) & 15];
            }
            cost += 3 * mk[2][j][k][(sg + 3 * a) & 15];
            cost += 2 * mk[3][j][k][(sg + RtGeom<D>::S0) & 15];
          }
          if (cost < bcost) { bcost = cost; bestc = sg; }
        }
        for (int o = 0; o < n; ++o) {
          const uint32_t w = occ[r * 4 + o];
          const int j = (w & 0xff) >> 1, k = (w >> 8) & 0xff, a = (w >> 16) & 3;
          for (int b = 0; b < NEN; ++b) {
            if (b == a) continue;
            ++mk[0][j][k][(bestc + 3 * b) & 15];
            ++mk[1][j][k][(bestc + RtGeom<D>::M0 + rt_pair<D>(a, b)) & 15];
          }
          ++mk[2][j][k][(bestc + 3 * a) & 15];
          ++mk[3][j][k][(bestc + RtGeom<D>::S0) & 15];
        }
        const int res = (rs_inv * bestc) & 15;         // slot residue of bank class bestc
        info[r] = (info[r] & 0xff) | (res + 16 * cls_cnt[bestc]) << 8;
        ++cls_cnt[bestc];
      }
    reinterpret_cast<int *>(blk)[0] = nslot;
    if (cnt) {  // FEM_RT_PLACE_DEBUG: modelled g_b-load wavefronts per half-warp, before / after
      int w0 = 0, w1 = 0;
      for (int j = 0; j < nn && j < 16; ++j) {
        const int best = s_best[j];
        if (!best) continue;
        const int sno = ndw[j].y & 0xff;
        const uint16_t *ej = en + j * L.es;
        for (int k = 0; k < best; ++k) {
          int c0[16], c1[16];
          for (int b = 0; b < 16; ++b) c0[b] = c1[b] = 0;
          for (int q = 0; q < sno; ++q) {
            const int e = ej[q * best + k], r = e & 1023, b = (e >> 12) & 3;
            if (r >= ue) continue;
            ++c0[(RS * r + 3 * b) & 15];
            ++c1[(RS * (info[r] >> 8) + 3 * b) & 15];
          }
          int m0 = 0, m1 = 0;
          for (int b = 0; b < 16; ++b) { m0 = max(m0, c0[b]); m1 = max(m1, c1[b]); }
          w0 += m0; w1 += m1;
        }
      }
      cnt[2 * t] = w0; cnt[2 * t + 1] = w1;
    }
  }
  __syncthreads();
  // remap the entries and move the element connectivity / phases to their slots (holes:
  // lc.x = 0xffff, skipped by the context phase)
  for (int j = 0; j < nn; ++j) {
    const int sno = ndw[j].y & 0xff;
    uint16_t *ej = en + j * L.es;
    for (int c = tid; c < L.es; c += nthr) {
      const int r = ej[c] & 1023;
      if (r < ue && (c < sno * (s_best[j] ? s_best[j] : 1) || !s_best[j]))
        ej[c] = (uint16_t)((ej[c] & ~1023) | (info[r] >> 8));
    }
  }
  ushort4 keep[4];
  uint8_t kph[4];
  for (int i = 0; i < 4; ++i) {
    const int r = tid + i * nthr;
    if (r < ue) {
      keep[i] = reinterpret_cast<const ushort4 *>(lc)[r];
      kph[i] = phase ? blk[L.off_ph + r] : 0;
    }
  }
  __syncthreads();
  for (int q = tid; q < nslot; q += nthr) reinterpret_cast<ushort4 *>(lc)[q] = make_ushort4(0xffff, 0, 0, 0);
  __syncthreads();
  for (int i = 0; i < 4; ++i) {
    const int r = tid + i * nthr;
    if (r < ue) {
      const int sl = info[r] >> 8;
      reinterpret_cast<ushort4 *>(lc)[sl] = keep[i];
      if (phase) blk[L.off_ph + sl] = kph[i];
    }
  }
}

// Node-tile plan over segments of a node list (the row form: one segment, the Morton order;
// the colored form, TR: one segment per node color, seeds in Morton order).  Tiles never
// straddle segments; segment g's tiles start at tile seg_tiles[g].
static fem_status build_tile_plan(Problem *p, const int32_t *order, const std::vector<int64_t> &seg,
                                  bool tr, RtPlan &out, cudaStream_t s) {
  const int D = p->dim, NEN = D + 1;
  const int64_t n = p->n_nodes;
  // max degree -> entry stride; max off-diagonal slots -> lanes per node
  std::vector<int64_t> hip(n + 1), hap(n + 1);
  FEM_CUDA(cudaMemcpyAsync(hip.data(), p->inc_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaMemcpyAsync(hap.data(), p->nadj_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  int IS = 0, SN = 0;
  for (int64_t i = 0; i < n; ++i) {
    IS = std::max<int>(IS, (int)(hip[i + 1] - hip[i]));
    SN = std::max<int>(SN, (int)(hap[i + 1] - hap[i]));
  }
  if (SN - 1 > kRtMaxSlots) return FEM_OK;
  // 8 lanes per node when the slots allow (2D Tri3: 6): 4 nodes per warp, 32-node tiles;
  // 16 lanes (3D Kuhn: 14 slots), 2 nodes per warp, kRtNT-node tiles; more slots
  // (unstructured meshes): 32 lanes, one node per warp, 8-node tiles (the element sets of
  // high-degree nodes are large), each lane summing slots ql, ql + 32
  const bool force32 = getenv("FEM_RT_LPN32") != nullptr;  // tests: the unstructured form anywhere
  const int LPN = force32 ? 32
                  : (D == 2 && SN - 1 <= 8 && !getenv("FEM_RT_LPN16")) ? 8
                  : (SN - 1 <= 16) ? 16 : 32;
  int NT = LPN == 8 ? 32 : LPN == 16 ? kRtNT : 8;
  // colored tiles: seeds of one color share no element, so a tile's element set is the union
  // of its seeds' stars (~24 per seed in 3D) — fewer seeds per tile keep the records small
  if (tr && FEM_CT_NT > 0) NT = std::min(NT, FEM_CT_NT);
  const int ng = (int)seg.size() - 1;
  out.seg_tiles.assign(ng + 1, 0);
  for (int g = 0; g < ng; ++g) out.seg_tiles[g + 1] = out.seg_tiles[g] + (seg[g + 1] - seg[g] + NT - 1) / NT;
  const int64_t nt = out.seg_tiles[ng];
  const int MS = std::max(LPN, SN - 1);  // slots per node the layout holds
  const int ES = std::max((((NEN - 1) * IS) + 7) & ~7, FEM_RT_SCHED ? MS * (D == 3 ? 7 : 5) : 0),
            SS = (MS + 1 + 3) & ~3;
  if (IS == 0 || ES > 65535 || nt == 0) return FEM_OK;
  int *d_bad = nullptr;
  int32_t *cnt = nullptr;
  FEM_CUDA(cudaMalloc(&d_bad, sizeof(int) * (2 + kRtSchedHist)));
  FEM_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int) * (2 + kRtSchedHist), s));
  FEM_CUDA(cudaMalloc(&cnt, sizeof(int32_t) * 2 * nt));
  FEM_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
  const bool dbg = getenv("FEM_RT_PLACE_DEBUG") != nullptr;
  auto plan = [&](const RtLayout &L, uint8_t *meta) -> fem_status {  // count (meta null) / fill
    for (int g = 0; g < ng; ++g) {
      const int64_t tiles = out.seg_tiles[g + 1] - out.seg_tiles[g];
      if (!tiles) continue;
      const int32_t *ord = order + seg[g];
      const int64_t cnt_n = seg[g + 1] - seg[g];
      int32_t *c = cnt + 2 * out.seg_tiles[g];
      uint8_t *m = meta ? meta + out.seg_tiles[g] * (int64_t)L.mb : nullptr;
      int32_t *cc = (meta && !dbg) ? nullptr : c;
      if (D == 2) k_rt_plan<2><<<(unsigned)tiles, 256, 0, s>>>(ord, cnt_n, p->inc_ptr, p->inc, p->conn, p->phase, p->nadj_ptr, p->nadj, p->row_ptr, p->node_bc, L, cc, m, d_bad);
      else k_rt_plan<3><<<(unsigned)tiles, 256, 0, s>>>(ord, cnt_n, p->inc_ptr, p->inc, p->conn, p->phase, p->nadj_ptr, p->nadj, p->row_ptr, p->node_bc, L, cc, m, d_bad);
      FEM_LAUNCH_CHECK("node-tile plan");
    }
    return FEM_OK;
  };
  // SoA records (FEM_RT_SOA): 3D row form with 16 lanes per <= 16-node tile; the environment
  // variable FEM_RT_SOA=0/1 overrides the compiled default at run time (A/B)
  const char *soa_env = getenv("FEM_RT_SOA");  // run-time override of the default (A/B)
  bool soa = (soa_env ? atoi(soa_env) != 0 : FEM_RT_SOA) && D == 3 && LPN == 16 && NT <= 16 &&
             !tr && !FEM_RT_PLACE && !getenv("FEM_RT_SOA_OFF");
  std::vector<int32_t> hc(2 * nt);
  int hbad = 0, uem = 0, unm = 0;
  for (int pass = 0; pass < 2; ++pass) {
    RtLayout L0 = rt_layout(NT, LPN, 8, 8, ES, SS, p->phase != nullptr, tr, soa);
    FEM_CUDA(cudaMemsetAsync(d_bad, 0, sizeof(int), s));
    fem_status st0 = plan(L0, nullptr);
    if (st0) return st0;
    FEM_CUDA(cudaMemcpyAsync(hc.data(), cnt, sizeof(int32_t) * 2 * nt, cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaMemcpyAsync(&hbad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaStreamSynchronize(s));
    uem = unm = 0;
    for (int64_t t = 0; t < nt; ++t) {
      uem = std::max(uem, hc[2 * t]);
      unm = std::max(unm, hc[2 * t + 1]);
    }
    if (!soa || (!hbad && uem <= kRtSoaS)) break;
    soa = false;  // a tile's colored records exceed the SoA stride: odd-stride records
  }
  uem = soa ? kRtSoaS : (uem + 7) & ~7;
  unm = (unm + 7) & ~7;
  const RtLayout L = rt_layout(NT, LPN, uem, unm, ES, SS, p->phase != nullptr, tr, soa);
  // shared memory of the assembly kernel: 3 metadata blocks, 2 node-data buffers, records
  const int RS = D == 3 ? RtGeom<3>::RS : RtGeom<2>::RS;
  const int BP = D == 3 ? RtGeom<3>::BP : RtGeom<2>::BP;
  const size_t recw = soa ? (size_t)kRtSoaF * kRtSoaS : (size_t)RS * (uem + 1);
  const size_t smem = 3 * (size_t)L.mb + 2 * sizeof(double) * 2 * D * (size_t)unm +
                      sizeof(double) * recw +
                      (FEM_RT_DIAG_SMEM ? sizeof(double) * (rt_threads(tr) / 32) * 32 * BP : 0);
  if (hbad || uem >= 1024 || smem > 220 * 1024) {
    cudaFree(d_bad); cudaFree(cnt);
    return FEM_OK;
  }
  FEM_CUDA(cudaMalloc(&out.meta, (size_t)L.mb * nt));
  fem_status st = plan(L, out.meta);
  if (st) return st;
  if (dbg) {
    std::vector<int32_t> hd(2 * nt);
    FEM_CUDA(cudaMemcpyAsync(hd.data(), cnt, sizeof(int32_t) * 2 * nt, cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaStreamSynchronize(s));
    long long a0 = 0, a1 = 0;
    for (int64_t q = 0; q < nt; ++q) { a0 += hd[2 * q]; a1 += hd[2 * q + 1]; }
    fprintf(stderr, "[rt place] modelled g_b wavefronts per half-warp step: identity %lld, placed %lld\n", a0, a1);
  }
  int hist[2 + kRtSchedHist];
  FEM_CUDA(cudaMemcpyAsync(hist, d_bad, sizeof(hist), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  hbad = hist[0];
  if (getenv("FEM_RT_SCHED_STATS")) {
    long long n = 0, w = 0;
    fprintf(stderr, "[rt plan] soa=%d tiles=%lld uem=%d schedule lengths:", L.soa, (long long)nt, L.uem);
    for (int c = 0; c <= kRtSchedHist; ++c)
      if (hist[1 + c]) {
        if (c == kRtSchedHist) fprintf(stderr, " grouped:%d", hist[1 + c]);
        else fprintf(stderr, " %d:%d", c, hist[1 + c]);
        if (c < kRtSchedHist) { n += hist[1 + c]; w += (long long)c * hist[1 + c]; }
      }
    fprintf(stderr, "  mean %.3f\n", n ? (double)w / n : 0.0);
  }
  cudaFree(d_bad);
  cudaFree(cnt);
  if (hbad) {
    cudaFree(out.meta);
    out.meta = nullptr;
    return FEM_OK;
  }
  out.ntiles = nt;
  int *l = out.layout;
  l[0] = L.nt; l[1] = L.uem; l[2] = L.unm; l[3] = L.es; l[4] = L.ss; l[5] = L.mb;
  l[6] = L.off_halo; l[7] = L.off_lc; l[8] = L.off_ph; l[9] = L.off_nd; l[10] = L.off_so;
  l[11] = L.off_sb; l[12] = L.off_en; l[13] = L.lpn; l[14] = L.off_tb; l[15] = L.off_tsn;
  l[16] = L.soa;
  out.smem = (int)smem;
  out.state = 1;
  return FEM_OK;
}

fem_status build_row_tiles(Problem *p, cudaStream_t s) {
  if (p->rt.state) return FEM_OK;
  p->rt.state = -1;
  if (p->n_nodes == 0 || p->n_elems == 0 || getenv("FEM_ROWS_PULL")) return FEM_OK;
  fem_status st = morton_node_order(p, s);
  if (st) return st;
  return build_tile_plan(p, p->node_order, {0, p->n_nodes}, false, p->rt, s);
}

// fused colored Alg. 2 on node tiles: one segment per node color (p->ncolor_list / ncolor_off)
fem_status build_colored_tiles(Problem *p, cudaStream_t s) {
  if (p->ct.state) return FEM_OK;
  p->ct.state = -1;
  if (p->n_nodes == 0 || p->n_elems == 0 || p->n_mpc || !p->ncolor_list || getenv("FEM_ROWS_PULL"))
    return FEM_OK;
  return build_tile_plan(p, p->ncolor_list, p->ncolor_off, true, p->ct, s);
}

// ------------------------------------------------------------------ kernel
__device__ __forceinline__ void rt_cp16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void rt_cp8(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void rt_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void rt_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

struct RtArgs {
  const uint8_t *meta;
  int64_t n_tiles;
  RtLayout L;
  const double *coords, *z;
  double lam, mu;
  const double *lam_tab, *mu_tab;
  int has_phase, bc;
  double *vals;
  int *err;
};

// TR: fused colored Alg. 2 (FEM_ASSEMBLE_COLORED, reading R13) on node tiles of one node color:
// each seed's column blocks K[m, n] = K[n, m]^T are written at their decompressed CSR slots
// (row m D + k, column n D + i), conflict-free within a color; the diagonal block as the row form.
template <int D, int MAT, int LPN, bool TR = false, bool SOA = false>
__global__ void __launch_bounds__(rt_threads(TR), TR ? FEM_CT_MINB : FEM_RT_MINB) k_rows_tile(RtArgs A) {
  constexpr int NTH = rt_threads(TR);
  using Gm = RtGeom<D>;
  constexpr int NEN = Gm::NEN, BS = Gm::BS, RS = Gm::RS;
  static_assert(!SOA || (D == 3 && LPN == 16 && !TR), "SoA records: 3D row form, 16 lanes");
  constexpr int S = kRtSoaS;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char sm_rt[];
  const RtLayout &L = A.L;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int mb = L.mb, unm = L.unm;
  unsigned char *metab = sm_rt;
  double *nodeb = reinterpret_cast<double *>(sm_rt + 3 * mb);  // [2][2][unm][D]: x | u
  double *rec = nodeb + 2 * 2 * unm * D;                         // [uem][RS]
  // AoS: [uem + 1][RS] (the last one the zero record of idle steps); SoA: [kRtSoaF][S]
  double *scratch = rec + (SOA ? (size_t)kRtSoaF * S : (size_t)(L.uem + 1) * RS);  // [8 warps][32][BP]
  if (!SOA)
    for (int q = tid; q < RS; q += NTH) rec[(size_t)L.uem * RS + q] = 0.0;  // zero record
  const int64_t G = gridDim.x;

  __shared__ __align__(8) uint64_t mb_meta[3];
  if (FEM_RT_TMA_META && tid == 0) {
    for (int b = 0; b < 3; ++b) mb_init(&mb_meta[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // metadata of tile t into buffer b: one bulk copy (FEM_RT_TMA_META) or 16-byte cp.async
  auto issue_meta = [&](int64_t t, int b) {
    const unsigned char *src = A.meta + t * (int64_t)mb;
    unsigned char *dst = metab + b * mb;
    if (FEM_RT_TMA_META) {
      if (tid == 0) {
        mb_expect_tx(&mb_meta[b], (unsigned)mb);
        bulk_g2s(dst, src, (unsigned)mb, &mb_meta[b]);
      }
    } else {
      for (int off = tid * 16; off < mb; off += NTH * 16) rt_cp16(dst + off, src + off);
    }
  };
  // wait for the metadata of the k-th tile of this CTA (buffer k % 3, use k / 3)
  auto wait_meta = [&](int k) {
    if (FEM_RT_TMA_META) mb_wait(&mb_meta[k % 3], (unsigned)(k / 3) & 1u);
  };
  auto issue_nodes = [&](const unsigned char *m, double *dst) {
    const int un = reinterpret_cast<const int *>(m)[1];
    const int32_t *hid = reinterpret_cast<const int32_t *>(m + L.off_halo);
    if (FEM_RT_ISSUE_NODE) {  // one thread per halo node: D copies of x and of z each
      for (int r = tid; r < un; r += NTH) {
        const int64_t g = (int64_t)hid[r] * D;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          rt_cp8(dst + r * D + c, A.coords + g + c);
          rt_cp8(dst + unm * D + r * D + c, A.z + g + c);
        }
      }
    } else {
      for (int i = tid; i < un * D; i += NTH) {
        const int64_t g = (int64_t)hid[i / D] * D + (i % D);
        rt_cp8(dst + i, A.coords + g);
        rt_cp8(dst + unm * D + i, A.z + g);
      }
    }
  };

  int64_t t = blockIdx.x;
  if (t < A.n_tiles) {
    issue_meta(t, 0);
    rt_commit();
    rt_wait_all();
    wait_meta(0);
    __syncthreads();
    issue_nodes(metab, nodeb);
    if (t + G < A.n_tiles) issue_meta(t + G, 1);
    rt_commit();
  }
  for (int k = 0; t < A.n_tiles; ++k, t += G) {
    rt_wait_all();
    __syncthreads();
    const unsigned char *m = metab + (k % 3) * mb;
    const double *xs = nodeb + (k & 1) * 2 * unm * D, *us = xs + unm * D;
    if (t + G < A.n_tiles) {
      wait_meta(k + 1);
      issue_nodes(metab + ((k + 1) % 3) * mb, nodeb + ((k + 1) & 1) * 2 * unm * D);
    }
    if (t + 2 * G < A.n_tiles) issue_meta(t + 2 * G, (k + 2) % 3);
    rt_commit();
    const int ue = reinterpret_cast<const int *>(m)[0];
    const int nn = reinterpret_cast<const int *>(m)[2];
    // ---- 1: element contexts
    const uint16_t *lc = reinterpret_cast<const uint16_t *>(m + L.off_lc);
    for (int e = tid; e < (FEM_RT_DIAG_SKIP == 1 ? 0 : ue); e += NTH) {
      const ushort4 l4 = reinterpret_cast<const ushort4 *>(lc)[e];
      if (l4.x == 0xffff) continue;  // placement hole (no entry reads it)
      const int li[4] = {l4.x, l4.y, l4.z, l4.w};
      double x[NEN][D], u[NEN][D], G[NEN][D], vol;
#pragma unroll
      for (int a = 0; a < NEN; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) {
          x[a][i] = xs[li[a] * D + i];
          u[a][i] = us[li[a] * D + i];
        }
#if FEM_RT_COF
      // cofactor form with the SFU-seeded reciprocal (reading R12): G_a = c_a / det (a >= 1),
      // G_0 = -sum_a G_a — no IEEE divisions and their slow-path branches
      double id0;
      const double det0 = cof_geometry<D>(x, G, id0);
      vol = det0 * (D == 3 ? 1.0 / 6.0 : 0.5);
#else
      const double det0 = geometry<D>(x, G, vol);
#endif
      double lam = A.lam, mu = A.mu;
      if (A.has_phase) {
        const int ph = m[L.off_ph + e];
        lam = A.lam_tab[ph];
        mu = A.mu_tab[ph];
      }
      // field f of this record: AoS r[f], SoA r[f * S]
      double *r = rec + (SOA ? e : e * RS);
      constexpr int FS = SOA ? S : 1;
      double c1 = mu;
      bool ok = true;
      if constexpr (MAT == FEM_LINEAR_ELASTIC) {
#pragma unroll
        for (int a = 0; a < NEN; ++a)
#pragma unroll
          for (int i = 0; i < D; ++i) r[(SOA ? a * D + i : Gm::G0 + a * Gm::GP + i) * FS] = G[a][i];
      } else {
        // g_a = F^-T G_a is the shape-function gradient in the deformed configuration, i.e.
        // the geometry of the element at x + u, and J = det F = det J(x + u) / det J(x): two
        // independent geometry chains instead of H -> F^-1 -> F^-T G (shorter dependencies)
        double xc[NEN][D], g[NEN][D];
        deformed_edges<D>(x, u, xc);
#if FEM_RT_COF
        double idc;
        const double Jd = cof_geometry<D>(xc, g, idc) * id0;
#else
        double volc;
        const double Jd = geometry<D>(xc, g, volc) / det0;
#endif
        ok = Jd > 0.0;
        if (!ok) atomicOr(A.err, ERRW_INVERTED);
        c1 = ok ? mu - lam * fem_log(Jd) : 0.0;
#pragma unroll
        for (int a = 0; a < NEN; ++a)
#pragma unroll
          for (int i = 0; i < D; ++i)
            r[(SOA ? a * D + i : Gm::G0 + a * Gm::GP + i) * FS] = ok ? g[a][i] : 0.0;
      }
      const double smu = ok ? vol * mu : 0.0;
#pragma unroll
      for (int a = 0; a < NEN; ++a)
#pragma unroll
        for (int b = a + 1; b < NEN; ++b) {
          double gg = 0.0;
#pragma unroll
          for (int j = 0; j < D; ++j) gg = fma(G[a][j], G[b][j], gg);
          r[(SOA ? rt_soa_m(a, b) : Gm::M0 + rt_pair<D>(a, b)) * FS] = smu * gg;
        }
      r[(SOA ? 15 : Gm::S0) * FS] = ok ? vol * c1 : 0.0;
      r[(SOA ? 19 : Gm::S0 + 1) * FS] = ok ? vol * lam : 0.0;
    }
    __syncthreads();
    // ---- 2: rows, LPN lanes per tile node (NPW nodes per warp)
    constexpr int NPW = 32 / LPN;
    const int h = lane / LPN, ql = lane % LPN;
    const int4 *ndw = reinterpret_cast<const int4 *>(m + L.off_nd);
    for (int j = NPW * w + h; j < (FEM_RT_DIAG_SKIP == 2 ? 0 : L.nt); j += NPW * (NTH / 32)) {
      const int4 nd = ndw[j];
      const int sno = nd.y & 0xff, sn = (nd.y >> 8) & 0xff, ds = (nd.y >> 16) & 0xff;
      const unsigned bcn = A.bc ? ((unsigned)nd.y >> 24) : 0u;
      const int64_t rp0 = (int64_t)(uint32_t)nd.z | ((int64_t)nd.w << 32);
      // start of row i relative to rp0: i D sn + multiplier columns of the earlier rows
      auto roff = [&](int i) -> int64_t {
        return (int64_t)i * D * sn + (i == 0 ? 0 : (i == 1 ? (nd.x & 0xffff) : ((unsigned)nd.x >> 16)));
      };
      const uint16_t *ent = reinterpret_cast<const uint16_t *>(m + L.off_en) + j * L.es;
      const uint16_t *sof = reinterpret_cast<const uint16_t *>(m + L.off_so) + j * L.ss;
      const bool live = j < nn;
      double dacc = 0.0;  // lanes ql < BS: diagonal entry, summed over the slot passes
      // slot passes: 8 / 16 lanes are chosen only when every node has <= LPN slots (one
      // pass); 32 lanes (one node per warp) loop over ceil(sno / 32) passes
      const int npass = LPN == 32 ? (sno + LPN - 1) / LPN : 1;
      for (int pass = 0; pass < npass; ++pass) {
      const int q = pass * LPN + ql;           // this lane's slot in this pass
      int lo = 0, hi = 0;
      if (q < sno) {
        lo = sof[q];
        hi = sof[q + 1];
      }
      double acc[BS];
#pragma unroll
      for (int q = 0; q < BS; ++q) acc[q] = 0.0;
      if constexpr (SOA) {
        // SoA records: every load one wavefront per half-warp (the plan's colored records and
        // color-distinct co-scheduled steps); idle steps (0xffff) load nothing
#pragma unroll kRtUnroll
        for (int c = lo; c < hi; ++c) {
          const uint32_t en = ent[c];
          if (en != 0xffffu) {
            const int rr = en & 1023u, a = (en >> 10) & 3u, b = (en >> 12) & 3u;
            const double *ra = rec + 3 * a * S + rr, *rb = rec + 3 * b * S + rr;
            const double Mab = rec[rt_soa_m(a, b) * S + rr];
            const double sc1 = rec[15 * S + rr], sc2 = rec[19 * S + rr];
            double ga[3], gb[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
              ga[i] = ra[i * S];
              gb[i] = rb[i * S];
            }
#pragma unroll
            for (int i = 0; i < D; ++i) {
              const double qi = sc2 * ga[i];
#pragma unroll
              for (int kk = 0; kk < D; ++kk) {
                double v = fma(sc1 * ga[kk], gb[i], acc[i * D + kk]);
                v = fma(qi, gb[kk], v);
                acc[i * D + kk] = (i == kk) ? v + Mab : v;
              }
            }
          }
        }
      } else
#pragma unroll kRtUnroll
      for (int c = lo; c < hi; ++c) {
        const uint32_t en = ent[c];
        const double *r = rec + (en & 1023u) * RS;
        const int a = (en >> 10) & 3u, b = (en >> 12) & 3u;
        double ga[Gm::GP + 1], gb[Gm::GP + 1];
        if constexpr (Gm::GP % 2 == 0 && Gm::RS % 2 == 0) {
#pragma unroll
          for (int i = 0; i < Gm::GP; i += 2) {
            const double2 x = *reinterpret_cast<const double2 *>(r + Gm::G0 + a * Gm::GP + i);
            const double2 y = *reinterpret_cast<const double2 *>(r + Gm::G0 + b * Gm::GP + i);
            ga[i] = x.x; ga[i + 1] = x.y;
            gb[i] = y.x; gb[i + 1] = y.y;
          }
        } else {
#pragma unroll
          for (int i = 0; i < D; ++i) {
            ga[i] = r[Gm::G0 + a * Gm::GP + i];
            gb[i] = r[Gm::G0 + b * Gm::GP + i];
          }
        }
        const double Mab = r[Gm::M0 + rt_pair<D>(a, b)];
        const double sc1 = r[Gm::S0], sc2 = r[Gm::S0 + 1];
#pragma unroll
        for (int i = 0; i < D; ++i) {
          const double qi = sc2 * ga[i];
#pragma unroll
          for (int kk = 0; kk < D; ++kk) {
            double v = fma(sc1 * ga[kk], gb[i], acc[i * D + kk]);
            v = fma(qi, gb[kk], v);
            acc[i * D + kk] = (i == kk) ? v + Mab : v;
          }
        }
      }
      if (TR && live && q < sno) {  // K[m D + k, n D + i] = K[n D + i, m D + k]
        const unsigned sbc = A.bc ? m[L.off_sb + j * L.ss + q] : 0u;
        const int64_t tb = reinterpret_cast<const int64_t *>(m + L.off_tb)[j * L.ss + q];
        const int snm = m[L.off_tsn + j * L.ss + q];
#pragma unroll
        for (int kk = 0; kk < D; ++kk) {
          double *row = A.vals + tb + (int64_t)kk * D * snm;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            double v = acc[i * D + kk];
            if ((sbc >> kk) & 1u) v = 0.0;   // identity row (m, kk), off-diagonal
            if ((bcn >> i) & 1u) v = 0.0;    // masked column (n, i)
            row[i] = v;
          }
        }
      }
      if (!TR && live && q < sno) {
        const unsigned sbc = A.bc ? m[L.off_sb + j * L.ss + q] : 0u;
        const int s = q + (q >= ds);
        double *row = A.vals + rp0 + s * D;
        if ((sbc | bcn) == 0u) {
#pragma unroll
          for (int i = 0; i < D; ++i)
#pragma unroll
            for (int kk = 0; kk < D; ++kk) row[roff(i) + kk] = acc[i * D + kk];
        } else {
#pragma unroll
          for (int i = 0; i < D; ++i)
#pragma unroll
            for (int kk = 0; kk < D; ++kk) {
              double v = acc[i * D + kk];
              if ((sbc >> kk) & 1u) v = 0.0;  // masked column
              if ((bcn >> i) & 1u) v = 0.0;   // identity row (off-diagonal)
              row[roff(i) + kk] = v;
            }
        }
      }
#if FEM_RT_DIAG_SMEM
      // diagonal block = -sum of the node's off-diagonal slots, ascending slot order
      double *scr = scratch + (w * 32 + lane) * Gm::BP;
#pragma unroll
      for (int qq = 0; qq < BS; ++qq) scr[qq] = acc[qq];
      __syncwarp();
      if (live && ql < BS) {
        const double *sb = scratch + (w * 32 + h * LPN) * Gm::BP + ql;
        const int cnt = min(LPN, sno - pass * LPN);
        if (FEM_RT_DIAG_UNROLL) {  // predicated, fully unrolled; even / odd slots in two chains
          double d0 = 0.0, d1 = 0.0;
#pragma unroll
          for (int qq = 0; qq < LPN; qq += 2) {
            if (qq < cnt) d0 += sb[qq * Gm::BP];
            if (qq + 1 < cnt) d1 += sb[(qq + 1) * Gm::BP];
          }
          dacc += d0 + d1;
        } else {
          for (int qq = 0; qq < cnt; ++qq) dacc += sb[qq * Gm::BP];
        }
      }
      __syncwarp();
      }  // slot passes
      if (live && ql < BS) {
        const int i = ql / D, kk = ql % D;
        double v = -dacc;
        if (bcn & (1u << kk)) v = 0.0;                      // masked column
        if (bcn & (1u << i)) v = (i == kk) ? 1.0 : 0.0;     // identity row
        A.vals[rp0 + roff(i) + ds * D + kk] = v;
      }
#else
      // diagonal block = -sum over the node's slots (fixed butterfly order)
#pragma unroll
      for (int q = 0; q < BS; ++q) {
        double v = acc[q];
#pragma unroll
        for (int o = LPN / 2; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o, LPN);
        acc[q] = v;
      }
      }  // slot passes (FEM_RT_DIAG_SMEM=0 supports one pass only: LPN >= slots)
      if (live) {
#pragma unroll
        for (int q = 0; q < BS; ++q)
          if (ql == q) {
            const int i = q / D, kk = q % D;
            double v = -acc[q];
            if (bcn & (1u << kk)) v = 0.0;                      // masked column
            if (bcn & (1u << i)) v = (i == kk) ? 1.0 : 0.0;     // identity row
            A.vals[rp0 + roff(i) + ds * D + kk] = v;
          }
      }
#endif
    }
  }
}

template <bool TR>
static fem_status launch_plan(Problem *p, const RtPlan &P, int64_t t0, int64_t tiles, const double *z,
                              double *vals, bool bc, cudaStream_t s) {
  RtArgs A{};
  const int *lay = P.layout;
  A.L.nt = lay[0]; A.L.uem = lay[1]; A.L.unm = lay[2]; A.L.es = lay[3]; A.L.ss = lay[4];
  A.L.mb = lay[5]; A.L.off_halo = lay[6]; A.L.off_lc = lay[7]; A.L.off_ph = lay[8];
  A.L.off_nd = lay[9]; A.L.off_so = lay[10]; A.L.off_sb = lay[11]; A.L.off_en = lay[12];
  A.L.lpn = lay[13]; A.L.off_tb = lay[14]; A.L.off_tsn = lay[15]; A.L.soa = lay[16];
  A.meta = P.meta + t0 * (int64_t)A.L.mb; A.n_tiles = tiles; A.coords = p->coords; A.z = z;
  A.lam = p->lam; A.mu = p->mu; A.lam_tab = p->lam_tab; A.mu_tab = p->mu_tab;
  A.has_phase = p->phase != nullptr; A.bc = bc ? 1 : 0; A.vals = vals; A.err = p->d_err;
  void (*kern)(RtArgs);
  const bool le = p->material == FEM_LINEAR_ELASTIC;
  const int lpn = A.L.lpn;
  if (p->dim == 2)
    kern = le ? (lpn == 8 ? k_rows_tile<2, FEM_LINEAR_ELASTIC, 8, TR> : lpn == 16 ? k_rows_tile<2, FEM_LINEAR_ELASTIC, 16, TR> : k_rows_tile<2, FEM_LINEAR_ELASTIC, 32, TR>)
              : (lpn == 8 ? k_rows_tile<2, FEM_NEO_HOOKEAN, 8, TR> : lpn == 16 ? k_rows_tile<2, FEM_NEO_HOOKEAN, 16, TR> : k_rows_tile<2, FEM_NEO_HOOKEAN, 32, TR>);
  else if (A.L.soa && !TR)
    kern = le ? k_rows_tile<3, FEM_LINEAR_ELASTIC, 16, false, true> : k_rows_tile<3, FEM_NEO_HOOKEAN, 16, false, true>;
  else
    kern = le ? (lpn == 16 ? k_rows_tile<3, FEM_LINEAR_ELASTIC, 16, TR> : k_rows_tile<3, FEM_LINEAR_ELASTIC, 32, TR>)
              : (lpn == 16 ? k_rows_tile<3, FEM_NEO_HOOKEAN, 16, TR> : k_rows_tile<3, FEM_NEO_HOOKEAN, 32, TR>);
  FEM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P.smem));
  int per_sm = 0;
  FEM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, rt_threads(TR), P.smem));
  int dev = 0, sms = 148;
  FEM_CUDA(cudaGetDevice(&dev));
  FEM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int64_t grid = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > tiles) grid = tiles;
  kern<<<(int)grid, rt_threads(TR), P.smem, s>>>(A);
  FEM_LAUNCH_CHECK("node-tile assembly");
  return FEM_OK;
}

fem_status launch_row_tiles(Problem *p, const double *z, double *vals, bool bc, cudaStream_t s) {
  return launch_plan<false>(p, p->rt, 0, p->rt.ntiles, z, vals, bc, s);
}

// one launch per node color (tiles of one color write disjoint slots)
fem_status launch_colored_tiles(Problem *p, const double *z, double *vals, bool bc, cudaStream_t s) {
  for (size_t g = 0; g + 1 < p->ct.seg_tiles.size(); ++g) {
    const int64_t tiles = p->ct.seg_tiles[g + 1] - p->ct.seg_tiles[g];
    if (!tiles) continue;
    fem_status st = launch_plan<true>(p, p->ct, p->ct.seg_tiles[g], tiles, z, vals, bc, s);
    if (st) return st;
  }
  return FEM_OK;
}

}  // namespace fem
