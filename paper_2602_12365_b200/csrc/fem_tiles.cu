// fem_tiles.cu — element tiles: the B200 form of Alg. 1's element batches.
//
// Setup: elements are ordered along a Morton curve of their centroids (cub radix sort) and
// cut into tiles of kTile = 256 consecutive elements — one CTA each.  Per tile a block
// radix sort of the tile's (node, element-slot) incidences yields the sorted list of the
// tile's unique nodes, the tile-local connectivity (uint16 indices into that list) and, per
// tile node, the list of its in-tile incidences; a node is "interior" when all of its
// incident elements lie in the tile.
//
// Element kernels (energy / residual / HVP): phase 0 stages the tile's nodal coordinates,
// u and v (masked at Dirichlet DOFs) in shared memory with coalesced loads of runs of
// consecutive nodes; phase 1 evaluates one element per thread from shared memory and writes
// its nodal contributions to a shared [slot][comp][element] array; phase 2 sums each tile
// node's in-tile incidences in a fixed order and writes the result: a plain store for
// interior nodes, one fp64 RED for nodes shared with other tiles (~1.8 REDs per DOF in 3D
// instead of 24 element-level atomics).  With FEM_DETERMINISTIC every tile-node sum goes to
// its own partial slot and a node-gather kernel adds the slots in tile order.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "element.cuh"
#include "fem_internal.cuh"
#include "pipe.cuh"

#ifndef FEM_PIPE_MINB2D
#define FEM_PIPE_MINB2D 0
#endif
#ifndef FEM_HVP_MINB
#define FEM_HVP_MINB 2
#endif
#ifndef FEM_RES_MINB
#define FEM_RES_MINB 3
#endif
#ifndef FEM_PIPE_MINB
#define FEM_PIPE_MINB 0  // 0: per-op choice (pipe_minb)
#endif
#ifndef FEM_PHASE2_SPLIT
#define FEM_PHASE2_SPLIT 0
#endif

#ifndef FEM_ELEM_SCHED
#define FEM_ELEM_SCHED 0  // A/B: 1 = slower (HVP 0.982 -> 1.013 ms at cfg 3)
#endif
#ifndef FEM_TILE_SCHED
#define FEM_TILE_SCHED 1
#endif
#ifndef FEM_RES_SPATIAL
#define FEM_RES_SPATIAL 1
#endif
#ifndef FEM_HVP_SPATIAL
#define FEM_HVP_SPATIAL 1
#endif
// Phase 2 as a balanced task schedule (k_build_sched) instead of one thread per tile node.
// A/B at cfg 3 (r02): HVP 0.975 -> 1.011 ms, residual 0.811 -> 0.811 ms: the barrier stall
// moves to shared-memory latency and the 5 KB of schedule per tile adds 0.3 GB of DRAM reads
// per launch, so the one-thread-per-node sums stay the default.
#ifndef FEM_P2_BAL
#define FEM_P2_BAL 0
#endif
// Phase 2 over padded incidence groups (k_g8_fill; A/B r02 at cfg 3: HVP 0.936 -> 0.923 ms,
// residual 0.807 -> 0.818 ms — within noise, so off by default): each node's list is padded to a multiple
// of 8 entries (pad = a zero column of the contribution array) and stored as precomputed
// contribution offsets, so a node thread loads 8 offsets with one 16-byte shared load and
// then issues 8 x D independent value loads: one dependent shared-memory round trip per 8
// incidences instead of two per 2 (the node sums were the kernels' longest dependency chain).
#ifndef FEM_P2_G8
#define FEM_P2_G8 0
#endif
// Phase 2 over a node-major contribution array (FEM_P2_NM): phase 1 stores element e's
// contribution for local node a at the position of incidence (e, a) in the node-sorted
// incidence list (lpos, setup), so each tile node sums a contiguous run cb[q D + c],
// q in [ptr[r], ptr[r+1]) — no index loads, no dependent address chain.  A/B r02 at cfg 3:
// HVP 0.935 -> 1.041 ms, residual 0.807 -> 0.928 ms (the scattered phase-1 stores conflict
// in the banks), so off by default.
#ifndef FEM_P2_NM
#define FEM_P2_NM 0
#endif
// Two lanes per tile node in phase 2 (FEM_P2_PAIR): A/B r02 at cfg 3 (same box): HVP 0.997 vs
// 0.938 ms, residual 0.864 vs 0.809 ms (the shuffles and the lost bank schedule cost more than
// the shorter per-node chains save), so off by default.
#ifndef FEM_P2_PAIR
#define FEM_P2_PAIR 0
#endif
// Phase-2 node order sorted by incidence count (FEM_P2_SORT): thread q of the node sums takes
// the tile node with the q-th longest list, so each warp's lanes loop about as often as its
// longest list and the short lists no longer idle in warps that hold a 24-incidence node.
// Parity-tested; A/B r02 at cfg 3: HVP 0.944 vs 0.909 ms (the warp of the longest lists is
// the critical path before the barrier either way, and the sorted groups lose the banks
// spread), so off by default.
#ifndef FEM_P2_SORT
#define FEM_P2_SORT 0
#endif
// unroll factor of the default node-sum loop (pairs of incidences per unrolled step)
// Phase-2 long-node split: nodes with more than FEM_P2_LSPLIT incidences are summed by two
// adjacent lanes (halves of the list; the even lane adds the odd lane's partial by one
// shuffle, fixed order), so the longest node-sum chain (24 incidences for an interior Kuhn
// node) halves while the other nodes keep one lane each and most warps stay free to start the
// next tile (two lanes for every node, FEM_P2_PAIR, kept all 8 warps busy: slower).  0 = off.
// Measured (r02, cfg 3, two A/B pairs): HVP 0.958 / 0.957 ms at threshold 12 (0.943 at 8,
// 0.957 at 16) against 0.923 / 0.922 off; residual 0.799 vs 0.793 — the extra phase-2 lanes
// cost more than the halved chains save.  Off; the task branch is compiled only when on.
#ifndef FEM_P2_LSPLIT
#define FEM_P2_LSPLIT 0
#endif
// Experiment (A/B only): phase 1 RED-adds each element's nodal contributions straight to the
// output (global fp64 atomics; the node data still staged per tile) and phase 2 is skipped —
// measures the price of global REDs against the tile reduction's node sums and barrier.
#ifndef FEM_P1_RED
#define FEM_P1_RED 0
#endif
// G8 node sums (padded groups of 8 incidence offsets, 16-byte loads) for the HVP kernels only,
// from a second metadata layout, the other operators keeping the default node sums.  Measured
// (r02, cfg 3, device-timed medians): G8 everywhere gave HVP 0.901 vs 0.924 ms but residual
// 0.842 vs 0.803 (the residual runs 3 CTAs/SM at 80 registers); HVP only: 0.902 / 0.903 vs
// 0.927 / 0.926 ms, residual unchanged; the linearized HVP stays on the default sums (G8:
// 0.961 vs 0.737 ms).
#ifndef FEM_WS  // warp-specialized tile kernels (k_tile_ws below)
#define FEM_WS 0
#endif
#ifndef FEM_HVP_G8
#define FEM_HVP_G8 1
#endif
#ifndef FEM_P2_UNROLL
#define FEM_P2_UNROLL 1
#endif
// Phase 0: one thread per tile node issues the node's D-vector copies (no div / mod by D;
// A/B r02: neutral, 0.975 vs 0.972 ms HVP)
// NH HVP in metric form (M_ab = c_a . c_b, D_ab = dv_b . cs_a): fewer FP64 operations than
// the dH / Ah products (tile_phase1)
#ifndef FEM_HVP_MD
#define FEM_HVP_MD 1
#endif
// node-data staging of the tile kernels: 1 = one thread per tile node (D copies of each
// array), 0 = one thread per component.  Re-measured on the end-of-round kernels (cfg 3,
// device-timed, two pairs): per component HVP 0.886 / 0.885 vs 0.899 / 0.901 ms, residual
// 0.785 / 0.785 vs 0.802 / 0.801, energy 0.378 / 0.379 vs 0.381 / 0.381 (was neutral in
// round 1): 0.
#ifndef FEM_ISSUE_NODE
#define FEM_ISSUE_NODE 0
#endif

namespace fem {

// row stride of the per-tile contribution array cb[(a D + c)][kCbStride]: G8 appends 8 zero
// columns (the pad entries of the incidence groups point there)
constexpr int kCbStride = FEM_P2_G8 ? kTile + 8 : kTile;
constexpr int kCbStrideG8 = kTile + 8;  // contribution rows of the G8 node sums (8 zero pad columns)
constexpr int kP2Unroll = FEM_P2_UNROLL;
static_assert(!(FEM_P2_G8 && FEM_P2_BAL), "FEM_P2_G8 and FEM_P2_BAL are alternatives");
static_assert(!(FEM_P2_NM && (FEM_P2_G8 || FEM_P2_BAL)), "FEM_P2_NM is an alternative phase 2");

// ------------------------------------------------------------------ setup
__global__ void k_bbox_partial(const double *coords, int64_t n, int dim, double *part) {
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int c = 0; c < dim; ++c) {
      const double x = coords[i * dim + c];
      lo[c] = fmin(lo[c], x);
      hi[c] = fmax(hi[c], x);
    }
  __shared__ double s[2][3][kThreads];
  for (int c = 0; c < 3; ++c) { s[0][c][threadIdx.x] = lo[c]; s[1][c][threadIdx.x] = hi[c]; }
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o)
      for (int c = 0; c < 3; ++c) {
        s[0][c][threadIdx.x] = fmin(s[0][c][threadIdx.x], s[0][c][threadIdx.x + o]);
        s[1][c][threadIdx.x] = fmax(s[1][c][threadIdx.x], s[1][c][threadIdx.x + o]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int c = 0; c < 3; ++c) {
      part[blockIdx.x * 6 + c] = s[0][c][0];
      part[blockIdx.x * 6 + 3 + c] = s[1][c][0];
    }
}

__device__ __forceinline__ uint64_t spread3(uint64_t x) {  // 21 bits -> every 3rd bit
  x &= 0x1fffff;
  x = (x | x << 32) & 0x1f00000000ffffull;
  x = (x | x << 16) & 0x1f0000ff0000ffull;
  x = (x | x << 8) & 0x100f00f00f00f00full;
  x = (x | x << 4) & 0x10c30c30c30c30c3ull;
  x = (x | x << 2) & 0x1249249249249249ull;
  return x;
}

__device__ __forceinline__ uint64_t spread2(uint64_t x) {  // 31 bits -> every 2nd bit
  x &= 0x7fffffffull;
  x = (x | x << 16) & 0x0000ffff0000ffffull;
  x = (x | x << 8) & 0x00ff00ff00ff00ffull;
  x = (x | x << 4) & 0x0f0f0f0f0f0f0f0full;
  x = (x | x << 2) & 0x3333333333333333ull;
  x = (x | x << 1) & 0x5555555555555555ull;
  return x;
}

template <int D>
__global__ void k_morton(const double *coords, const int32_t *conn, int64_t E, double3 lo,
                         double3 scale, uint64_t *keys, int32_t *idx, int32_t *node_cnt) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (int64_t)gridDim.x * blockDim.x) {
    double c[3] = {0, 0, 0};
    for (int a = 0; a < D + 1; ++a) {
      const int32_t n = conn[e * (D + 1) + a];
      atomicAdd(node_cnt + n, 1);
      for (int i = 0; i < D; ++i) c[i] += coords[(int64_t)n * D + i];
    }
    const double l[3] = {lo.x, lo.y, lo.z}, s[3] = {scale.x, scale.y, scale.z};
    uint64_t q[3];
    for (int i = 0; i < D; ++i) {
      double t = (c[i] / (D + 1) - l[i]) * s[i];
      q[i] = (uint64_t)fmax(0.0, t);
    }
    keys[e] = (D == 3) ? (spread3(q[0]) | spread3(q[1]) << 1 | spread3(q[2]) << 2)
                       : (spread2(q[0]) | spread2(q[1]) << 1);
    idx[e] = (int32_t)e;
  }
}

template <int D>
__global__ void __launch_bounds__(kTile) k_tile_build(const int32_t *conn, const int32_t *perm,
                                                      int64_t E, const int32_t *node_cnt,
                                                      TileSet T) {
  constexpr int ITEMS = D + 1;
  constexpr int MAXE = kTile * ITEMS;
  using Sort = cub::BlockRadixSort<int32_t, kTile, ITEMS, uint16_t>;
  using Scan = cub::BlockScan<int, kTile>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ int32_t s_keys[MAXE + 1];
  __shared__ int s_U, s_valid;
  const int t = blockIdx.x, tid = threadIdx.x;
  int32_t keys[ITEMS];
  uint16_t vals[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int pos = tid * ITEMS + i;
    const int el = pos / (D + 1), a = pos % (D + 1);
    const int64_t eg = (int64_t)t * kTile + el;
    if (eg < E) {
      keys[i] = conn[(int64_t)perm[eg] * (D + 1) + a];
      vals[i] = (uint16_t)(el * 4 + a);
    } else {
      keys[i] = INT32_MAX;
      vals[i] = 0xffff;
    }
  }
  Sort(tmp.sort).Sort(keys, vals);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) s_keys[tid * ITEMS + i] = keys[i];
  __syncthreads();
  int head[ITEMS], nh = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int pos = tid * ITEMS + i;
    head[i] = keys[i] != INT32_MAX && (pos == 0 || s_keys[pos - 1] != keys[i]);
    nh += head[i];
  }
  int base = 0, total = 0;
  Scan(tmp.scan).ExclusiveSum(nh, base, total);
  const int64_t toff = (int64_t)t * MAXE;
  int rank = base - 1;
  int valid = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int pos = tid * ITEMS + i;
    if (keys[i] == INT32_MAX) continue;
    ++valid;
    rank += head[i];
    T.inc[toff + pos] = vals[i];
    const int el = vals[i] >> 2, a = vals[i] & 3;
    T.lconn[((int64_t)t * kTile + el) * 4 + a] = (uint16_t)rank;
    if (head[i]) {
      T.nodes[toff + rank] = keys[i];
      T.ptr[(int64_t)t * (MAXE + 1) + rank] = (uint16_t)pos;
    }
  }
  if (tid == 0) s_valid = 0;
  __syncthreads();
  atomicAdd(&s_valid, valid);
  if (tid == 0) s_U = total;
  __syncthreads();
  if (tid == 0) {
    T.U[t] = total;
    T.ptr[(int64_t)t * (MAXE + 1) + total] = (uint16_t)s_valid;
  }
  __syncthreads();
  for (int r = tid; r < s_U; r += kTile) {
    const int lo = T.ptr[(int64_t)t * (MAXE + 1) + r];
    const int hi = (r + 1 < s_U) ? T.ptr[(int64_t)t * (MAXE + 1) + r + 1] : s_valid;
    T.interior[toff + r] = (hi - lo) == node_cnt[T.nodes[toff + r]];
  }
  if (D == 2) {  // pad slot 3 of the tile-local connectivity
    const int64_t e = (int64_t)t * kTile + tid;
    T.lconn[e * 4 + 3] = 0;
  }
}

// Phase-1 bank scheduling (FEM_ELEM_SCHED): thread tid of a tile reads the D-vectors of its
// element's nodes at nodal-buffer offsets D lconn[a] (+ i), bank (D lconn[a] + i) mod 16.
// Reorder the elements inside each tile (greedy, warp by warp: the element among the next
// kSchedWin unplaced ones whose NEN banks the warp uses least) so a warp's node reads spread
// over the banks.  The tile's element set, and with it every per-tile structure, is unchanged.
constexpr int kSchedWin = 32;
template <int D>
__global__ void k_sched_elems(const uint16_t *lconn, int32_t *perm, int64_t E, int64_t nt) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const int64_t e0 = t * kTile;
  const int n = (int)(E - e0 < kTile ? E - e0 : kTile);
  uint32_t taken[kTile / 32];
  for (int q = 0; q < kTile / 32; ++q) taken[q] = 0;
  uint16_t order[kTile];
  int first = 0;
  for (int w = 0; w * 32 < n; ++w) {
    uint8_t cnt[D + 1][16];
    for (int a = 0; a <= D; ++a)
      for (int b = 0; b < 16; ++b) cnt[a][b] = 0;
    for (int l = 0; l < 32 && w * 32 + l < n; ++l) {
      while ((taken[first >> 5] >> (first & 31)) & 1u) ++first;
      int best = first, bc = 1 << 30, seen = 0;
      for (int q = first; q < n && seen < kSchedWin && bc > 0; ++q) {
        if ((taken[q >> 5] >> (q & 31)) & 1u) continue;
        ++seen;
        int c = 0;
        for (int a = 0; a <= D; ++a) c += cnt[a][(D * lconn[(e0 + q) * 4 + a]) & 15];
        if (c < bc) { bc = c; best = q; }
      }
      taken[best >> 5] |= 1u << (best & 31);
      for (int a = 0; a <= D; ++a) ++cnt[a][(D * lconn[(e0 + best) * 4 + a]) & 15];
      order[w * 32 + l] = (uint16_t)best;
    }
  }
  int32_t pv[kTile];
  for (int q = 0; q < n; ++q) pv[q] = perm[e0 + order[q]];
  for (int q = 0; q < n; ++q) perm[e0 + q] = pv[q];
}

__global__ void k_permute_u8(const uint8_t *src, const int32_t *perm, int64_t n, uint8_t *dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}

__global__ void k_histogram64(const int32_t *keys, int64_t n, int64_t *cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long *>(cnt + keys[i]), 1ull);
}

// deterministic mode: node -> partial slots (tile order)
__global__ void k_slot_pairs(TileSet T, int64_t n_tiles, const int64_t *slot_off, int32_t *key,
                             int32_t *val) {
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const int U = T.U[t];
    for (int r = threadIdx.x; r < U; r += blockDim.x) {
      key[slot_off[t] + r] = T.nodes[t * T.maxe + r];
      val[slot_off[t] + r] = (int32_t)(slot_off[t] + r);
    }
  }
}

fem_status pack_tile_meta(Problem *p, cudaStream_t s);

fem_status build_tiles(Problem *p, cudaStream_t s) {
  TileSet &T = p->tiles;
  if (T.built || p->n_elems == 0) return FEM_OK;
  const int D = p->dim;
  const int64_t E = p->n_elems;
  const int maxe = kTile * (D + 1);
  T.maxe = maxe;
  T.n_tiles = (E + kTile - 1) / kTile;
  // bounding box
  const int nb = grid_for(p->n_nodes, kThreads, 256);
  double *part = nullptr;
  FEM_CUDA(cudaMalloc(&part, sizeof(double) * nb * 6));
  k_bbox_partial<<<nb, kThreads, 0, s>>>(p->coords, p->n_nodes, D, part);
  std::vector<double> hp(nb * 6);
  FEM_CUDA(cudaMemcpyAsync(hp.data(), part, sizeof(double) * nb * 6, cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  cudaFree(part);
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int b = 0; b < nb; ++b)
    for (int c = 0; c < 3; ++c) {
      lo[c] = std::min(lo[c], hp[b * 6 + c]);
      hi[c] = std::max(hi[c], hp[b * 6 + 3 + c]);
    }
  const double qmax = (D == 3) ? double((1 << 21) - 1) : double((1u << 31) - 1);
  double sc[3];
  for (int c = 0; c < 3; ++c) sc[c] = (c < D && hi[c] > lo[c]) ? qmax / (hi[c] - lo[c]) : 0.0;
  // Morton keys + stable sort
  uint64_t *keys = nullptr, *keys_out = nullptr;
  int32_t *idx = nullptr, *node_cnt = nullptr;
  FEM_CUDA(cudaMalloc(&keys, sizeof(uint64_t) * E));
  FEM_CUDA(cudaMalloc(&keys_out, sizeof(uint64_t) * E));
  FEM_CUDA(cudaMalloc(&idx, sizeof(int32_t) * E));
  FEM_CUDA(cudaMalloc(&node_cnt, sizeof(int32_t) * p->n_nodes));
  FEM_CUDA(cudaMalloc(&T.perm, sizeof(int32_t) * E));
  FEM_CUDA(cudaMemsetAsync(node_cnt, 0, sizeof(int32_t) * p->n_nodes, s));
  const double3 dlo = make_double3(lo[0], lo[1], lo[2]);
  const double3 dsc = make_double3(sc[0], sc[1], sc[2]);
  if (D == 3) k_morton<3><<<grid_for(E), kThreads, 0, s>>>(p->coords, p->conn, E, dlo, dsc, keys, idx, node_cnt);
  else k_morton<2><<<grid_for(E), kThreads, 0, s>>>(p->coords, p->conn, E, dlo, dsc, keys, idx, node_cnt);
  FEM_LAUNCH_CHECK("morton");
  size_t bytes = 0;
  FEM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys_out, idx, T.perm, (int)E, 0,
                                           64, s));
  fem_status st = ensure(p->tmp, bytes);
  if (st) return st;
  FEM_CUDA(cub::DeviceRadixSort::SortPairs(p->tmp.ptr, bytes, keys, keys_out, idx, T.perm, (int)E,
                                           0, 64, s));
  // tiles
  const int64_t nt = T.n_tiles;
  FEM_CUDA(cudaMalloc(&T.nodes, sizeof(int32_t) * nt * maxe));
  FEM_CUDA(cudaMalloc(&T.U, sizeof(int32_t) * nt));
  FEM_CUDA(cudaMalloc(&T.ptr, sizeof(uint16_t) * nt * (maxe + 1)));
  FEM_CUDA(cudaMalloc(&T.inc, sizeof(uint16_t) * nt * maxe));
  FEM_CUDA(cudaMalloc(&T.lconn, sizeof(uint16_t) * nt * kTile * 4));
  FEM_CUDA(cudaMalloc(&T.interior, sizeof(uint8_t) * nt * maxe));
  FEM_CUDA(cudaMemsetAsync(T.lconn, 0, sizeof(uint16_t) * nt * kTile * 4, s));
  if (D == 3) k_tile_build<3><<<(unsigned)nt, kTile, 0, s>>>(p->conn, T.perm, E, node_cnt, T);
  else k_tile_build<2><<<(unsigned)nt, kTile, 0, s>>>(p->conn, T.perm, E, node_cnt, T);
  FEM_LAUNCH_CHECK("tile build");
  if (FEM_ELEM_SCHED) {  // reorder inside the tiles, then rebuild the per-tile structures
    const unsigned g = (unsigned)((nt + 63) / 64);
    if (D == 3) k_sched_elems<3><<<g, 64, 0, s>>>(T.lconn, T.perm, E, nt);
    else k_sched_elems<2><<<g, 64, 0, s>>>(T.lconn, T.perm, E, nt);
    FEM_CUDA(cudaMemsetAsync(T.lconn, 0, sizeof(uint16_t) * nt * kTile * 4, s));
    if (D == 3) k_tile_build<3><<<(unsigned)nt, kTile, 0, s>>>(p->conn, T.perm, E, node_cnt, T);
    else k_tile_build<2><<<(unsigned)nt, kTile, 0, s>>>(p->conn, T.perm, E, node_cnt, T);
    FEM_LAUNCH_CHECK("tile element scheduling");
  }
  if (p->phase) {
    FEM_CUDA(cudaMalloc(&T.phase, E));
    k_permute_u8<<<grid_for(E), kThreads, 0, s>>>(p->phase, T.perm, E, T.phase);
  }
  // max U (smem sizing) and slot offsets for the deterministic mode
  std::vector<int32_t> hU(nt);
  FEM_CUDA(cudaMemcpyAsync(hU.data(), T.U, sizeof(int32_t) * nt, cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  T.max_U = 0;
  std::vector<int64_t> off(nt + 1, 0);
  for (int64_t t = 0; t < nt; ++t) {
    T.max_U = std::max(T.max_U, hU[t]);
    off[t + 1] = off[t] + hU[t];
  }
  T.n_slots = off[nt];
  FEM_CUDA(cudaMalloc(&T.slot_off, sizeof(int64_t) * (nt + 1)));
  FEM_CUDA(cudaMemcpyAsync(T.slot_off, off.data(), sizeof(int64_t) * (nt + 1), cudaMemcpyHostToDevice, s));
  // node -> slots CSR (stable by tile order)
  {
    int32_t *k_in = nullptr, *v_in = nullptr, *k_out = nullptr;
    FEM_CUDA(cudaMalloc(&k_in, sizeof(int32_t) * T.n_slots));
    FEM_CUDA(cudaMalloc(&v_in, sizeof(int32_t) * T.n_slots));
    FEM_CUDA(cudaMalloc(&k_out, sizeof(int32_t) * T.n_slots));
    FEM_CUDA(cudaMalloc(&T.node_slots, sizeof(int32_t) * T.n_slots));
    FEM_CUDA(cudaMalloc(&T.node_slot_ptr, sizeof(int64_t) * (p->n_nodes + 1)));
    k_slot_pairs<<<grid_for(nt * 64, 64, 148 * 64), 64, 0, s>>>(T, nt, T.slot_off, k_in, v_in);
    int bits = 1;
    while ((int64_t(1) << bits) < p->n_nodes) ++bits;
    size_t b2 = 0;
    FEM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b2, k_in, k_out, v_in, T.node_slots,
                                             (int)T.n_slots, 0, bits, s));
    st = ensure(p->tmp, b2);
    if (st) return st;
    FEM_CUDA(cub::DeviceRadixSort::SortPairs(p->tmp.ptr, b2, k_in, k_out, v_in, T.node_slots,
                                             (int)T.n_slots, 0, bits, s));
    // node_cnt of slots via histogram of k_out -> exclusive scan
    int64_t *c64 = nullptr;
    FEM_CUDA(cudaMalloc(&c64, sizeof(int64_t) * (p->n_nodes + 1)));
    FEM_CUDA(cudaMemsetAsync(c64, 0, sizeof(int64_t) * (p->n_nodes + 1), s));
    k_histogram64<<<grid_for(T.n_slots), kThreads, 0, s>>>(k_out, T.n_slots, c64);
    size_t b3 = 0;
    FEM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, b3, c64, T.node_slot_ptr, p->n_nodes + 1, s));
    st = ensure(p->tmp, b3);
    if (st) return st;
    FEM_CUDA(cub::DeviceScan::ExclusiveSum(p->tmp.ptr, b3, c64, T.node_slot_ptr, p->n_nodes + 1, s));
    FEM_CUDA(cudaStreamSynchronize(s));
    cudaFree(k_in); cudaFree(v_in); cudaFree(k_out); cudaFree(c64);
  }
  FEM_CUDA(cudaStreamSynchronize(s));
  cudaFree(keys); cudaFree(keys_out); cudaFree(idx); cudaFree(node_cnt);
  FEM_CUDA(cudaMalloc(&T.epart, sizeof(double) * nt));
  st = pack_tile_meta(p, s);
  if (st) return st;
  FEM_CUDA(cudaStreamSynchronize(s));
  T.built = true;
  return FEM_OK;
}

// ------------------------------------------------------------------ packed tile metadata
// Per tile one contiguous, 16-byte aligned block (copied into shared memory with 16-byte
// cp.async): header {U, n_valid}, nodes int32[um], lconn uint16[kTile][4], ptr
// uint16[um+1], inc uint16[kTile*4], interior uint8[um], bc uint8[um] (Dirichlet bits of
// each tile node), phase uint8[kTile] (optional).
static inline int round_up(int x, int m) { return (x + m - 1) / m * m; }

template <int D>
__global__ void k_pack_meta(TileSet T, const uint8_t *node_bc, int64_t E) {
  const int64_t t = blockIdx.x;
  uint8_t *base = T.meta + t * T.mb;
  const int U = T.U[t];
  const int64_t e0 = t * kTile;
  const int nvalid = (int)((E - e0 < kTile ? E - e0 : kTile) * (D + 1));
  if (threadIdx.x == 0) {
    reinterpret_cast<int *>(base)[0] = U;
    reinterpret_cast<int *>(base)[1] = nvalid;
    reinterpret_cast<int *>(base)[2] = T.shdr ? (int)T.shdr[t] : 0;
    reinterpret_cast<int *>(base)[3] = T.p2n ? T.p2n[t] : 0;  // phase-2 tasks (FEM_P2_LSPLIT)
  }
  if (T.shdr) {
    const int cap = T.sched_rounds * kTile;
    uint16_t *so = reinterpret_cast<uint16_t *>(base + T.off_soff);
    uint32_t *sm = reinterpret_cast<uint32_t *>(base + T.off_smeta);
    for (int i = threadIdx.x; i < cap * 8; i += blockDim.x) so[i] = T.soff[t * cap * 8 + i];
    for (int i = threadIdx.x; i < cap; i += blockDim.x) sm[i] = T.smeta[t * cap + i];
  }
  int32_t *nodes = reinterpret_cast<int32_t *>(base + T.off_nodes);
  for (int i = threadIdx.x; i < T.um; i += blockDim.x) nodes[i] = i < U ? T.nodes[t * T.maxe + i] : 0;
  uint16_t *lc = reinterpret_cast<uint16_t *>(base + T.off_lconn);
  for (int i = threadIdx.x; i < kTile * 4; i += blockDim.x) lc[i] = T.lconn[t * kTile * 4 + i];
  if (T.inc8) {
    uint16_t *ptr = reinterpret_cast<uint16_t *>(base + T.off_ptr);
    for (int i = threadIdx.x; i <= T.um; i += blockDim.x) ptr[i] = T.ptr8[t * (T.um + 1) + i];
    uint16_t *inc = reinterpret_cast<uint16_t *>(base + T.off_inc);
    for (int i = threadIdx.x; i < T.me8; i += blockDim.x) inc[i] = T.inc8[t * (int64_t)T.me8 + i];
  } else if (T.off_ptr >= 0) {
    uint16_t *ptr = reinterpret_cast<uint16_t *>(base + T.off_ptr);
    for (int i = threadIdx.x; i <= T.um; i += blockDim.x)
      ptr[i] = i <= U ? T.ptr[t * (T.maxe + 1) + i] : (uint16_t)nvalid;
    uint16_t *inc = reinterpret_cast<uint16_t *>(base + T.off_inc);
    if (FEM_P2_NM) {  // lpos[e 4 + a] = list position of incidence (e, a)
      for (int i = threadIdx.x; i < kTile * 4; i += blockDim.x) inc[i] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < nvalid; i += blockDim.x) inc[T.inc[t * T.maxe + i]] = (uint16_t)i;
    } else {
      // contribution offsets (a D kTile + el) of the incidences (el << 2 | a): the node sums
      // add cb[w + c kTile] without unpacking; the bank (el mod 16) is w mod 16 as before
      for (int i = threadIdx.x; i < kTile * 4; i += blockDim.x) {
        const int e = i < nvalid ? T.inc[t * T.maxe + i] : 0;
        inc[i] = (uint16_t)((e & 3) * D * kTile + (e >> 2));
      }
    }
  }
  for (int i = threadIdx.x; i < T.um; i += blockDim.x) {
    base[T.off_int + i] = i < U ? T.interior[t * T.maxe + i] : 0;
    base[T.off_bc + i] = i < U ? node_bc[T.nodes[t * T.maxe + i]] : 0;
  }
  if (T.phase)
    for (int i = threadIdx.x; i < kTile; i += blockDim.x)
      base[T.off_ph + i] = (e0 + i < E) ? T.phase[e0 + i] : 0;
  if (T.p2perm) {
    uint16_t *pp = reinterpret_cast<uint16_t *>(base + T.off_perm);
    const int n = T.p2n ? T.p2n[t] : U;
    for (int i = threadIdx.x; i < T.pcap; i += blockDim.x) pp[i] = i < n ? T.p2perm[t * T.maxe + i] : 0;
  }
}

// Phase-2 bank scheduling (FEM_TILE_SCHED): every tile node sums its incident contributions
// cb[(a D + c) kTile + el] in the order of its incidence list, and the 32 nodes of a warp step
// through their lists together; the shared-memory bank of a read is el mod 16 (64-bit words).
// Reorder each list (step by step, greedy: the remaining entry whose bank the warp's other
// nodes use least at this step) so a step's reads spread over the banks.  Only the (fixed,
// deterministic) summation order of each node changes.
__global__ void k_sched_inc(TileSet T) {
  const int64_t t = blockIdx.x;
  const int U = T.U[t];
  const uint16_t *ptr = T.ptr + t * (T.maxe + 1);
  uint16_t *inc = T.inc + t * T.maxe;
  const uint16_t *perm = T.p2perm ? T.p2perm + t * T.maxe : nullptr;  // phase-2 thread order
  for (int g = threadIdx.x; g * 32 < U; g += blockDim.x) {
    const int q0 = g * 32, q1 = min(U, q0 + 32);
    int len = 0;
    for (int q = q0; q < q1; ++q) {
      const int r = perm ? perm[q] : q;
      len = max(len, (int)ptr[r + 1] - (int)ptr[r]);
    }
    for (int w = 0; w < len; ++w) {
      // a warp's 64-bit shared loads are served per half-warp: banks must differ within each
      // group of 16 consecutive phase-2 threads
      int cnt[16];
      for (int qq = q0; qq < q1; ++qq) {
        if (((qq - q0) & 15) == 0)
          for (int b = 0; b < 16; ++b) cnt[b] = 0;
        const int r = perm ? perm[qq] : qq;
        const int lo = ptr[r] + w, hi = ptr[r + 1];
        if (lo >= hi) continue;
        int best = lo, bc = 1 << 30;
        for (int q = lo; q < hi && bc > 0; ++q) {
          const int c = cnt[(inc[q] >> 2) & 15];
          if (c < bc) { bc = c; best = q; }
        }
        const uint16_t x = inc[best];
        inc[best] = inc[lo];
        inc[lo] = x;
        ++cnt[(x >> 2) & 15];
      }
    }
  }
}

// Phase-2 thread order (FEM_P2_SORT): tile nodes by descending incidence count, ties in node
// order (counting sort per tile, one thread per tile).
__global__ void k_p2_perm(TileSet T) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T.n_tiles) return;
  const int U = T.U[t];
  const uint16_t *ptr = T.ptr + t * (T.maxe + 1);
  uint16_t *perm = T.p2perm + t * T.maxe;
  int maxlen = 0;
  for (int r = 0; r < U; ++r) maxlen = max(maxlen, (int)ptr[r + 1] - (int)ptr[r]);
  int pos = 0;
  for (int len = maxlen; len >= 0; --len)
    for (int r = 0; r < U; ++r)
      if ((int)ptr[r + 1] - (int)ptr[r] == len) perm[pos++] = (uint16_t)r;
}

// Phase-2 tasks (FEM_P2_LSPLIT): long nodes first as (first half, second half) lane pairs at
// even positions, then the other nodes in node order; entry = r | 1 << 14 (first half) | 1 << 15
// (second half).  One thread per tile.
__global__ void k_p2_tasks(TileSet T, int th) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T.n_tiles) return;
  const int U = T.U[t];
  const uint16_t *ptr = T.ptr + t * (T.maxe + 1);
  uint16_t *task = T.p2perm + t * T.maxe;
  int pos = 0;
  for (int r = 0; r < U; ++r)
    if ((int)ptr[r + 1] - (int)ptr[r] > th) {
      task[pos++] = (uint16_t)(r | 1 << 14);
      task[pos++] = (uint16_t)(r | 1 << 15);
    }
  for (int r = 0; r < U; ++r)
    if ((int)ptr[r + 1] - (int)ptr[r] <= th) task[pos++] = (uint16_t)r;
  T.p2n[t] = pos;
}

// Balanced phase-2 schedule (FEM_P2_BAL).  The tile's incidences (node r, element el, slot
// a) are cut into tasks of <= K incidences of one node (K in 4..8, the smallest that fits the
// lanes: rounds x kTile task slots), a node's g tasks on consecutive lanes of one warp; lane
// l sums its task's <= 8 contributions cb[(a D + c) kTile + el] (offsets w = a D kTile + el
// precomputed) for c < D, and the g lanes of a node combine by a shuffle tree (head = pos 0).
// Every thread of the CTA takes part, the longest chain is K loads instead of the node's
// full incidence count, and no address arithmetic runs per incidence.  The entries of each
// lane are ordered so that the 16 lanes of a half-warp hit distinct banks (el mod 16) at every
// step where possible.  Summation order is fixed by the schedule (deterministic).
__device__ int sched_lanes(const uint16_t *ptr, int U, int K) {
  int lane = 0;
  for (int r = 0; r < U; ++r) {
    const int n = ptr[r + 1] - ptr[r];
    const int g = (n + K - 1) / K;
    if ((lane & 31) + g > 32) lane = (lane + 31) & ~31;
    lane += g;
  }
  return lane;
}

__global__ void k_sched_count(TileSet T, int *max_lanes) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T.n_tiles) return;
  atomicMax(max_lanes, sched_lanes(T.ptr + t * (T.maxe + 1), T.U[t], 8));
}

template <int D>
__global__ void k_build_sched(TileSet T, int rounds) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T.n_tiles) return;
  const int U = T.U[t];
  const uint16_t *ptr = T.ptr + t * (T.maxe + 1);
  const uint16_t *inc = T.inc + t * T.maxe;
  const int cap = rounds * kTile;
  int K = 4;
  while (K < 8 && sched_lanes(ptr, U, K) > cap) ++K;
  uint16_t *so = T.soff + t * (int64_t)cap * 8;
  uint32_t *sm = T.smeta + t * (int64_t)cap;
  for (int j = 0; j < cap; ++j) {
    sm[j] = 0u;
    for (int q = 0; q < 8; ++q) so[j * 8 + q] = 0;
  }
  int lane = 0, gmax = 1;
  for (int r = 0; r < U; ++r) {
    const int lo = ptr[r], n = ptr[r + 1] - lo;
    const int g = (n + K - 1) / K;
    if ((lane & 31) + g > 32) lane = (lane + 31) & ~31;
    const int base = n / g, rem = n % g;
    int q0 = lo;
    for (int p = 0; p < g; ++p) {
      const int cnt = base + (p < rem ? 1 : 0);
      for (int q = 0; q < cnt; ++q) {
        const int e = inc[q0 + q];
        so[(lane + p) * 8 + q] = (uint16_t)((e & 3) * D * kTile + (e >> 2));
      }
      sm[lane + p] = (uint32_t)r | (uint32_t)cnt << 11 | (uint32_t)p << 15 | (uint32_t)g << 23;
      q0 += cnt;
    }
    lane += g;
    gmax = max(gmax, g);
  }
  for (int h = 0; h < cap / 16; ++h)        // bank order per half-warp and step
    for (int q = 0; q < 8; ++q) {
      int cnt[16];
      for (int b = 0; b < 16; ++b) cnt[b] = 0;
      for (int l = h * 16; l < h * 16 + 16; ++l) {
        const int n = (sm[l] >> 11) & 15;
        if (q >= n) continue;
        int best = q, bc = 1 << 30;
        for (int qq = q; qq < n && bc > 0; ++qq) {
          const int c = cnt[so[l * 8 + qq] & 15];
          if (c < bc) { bc = c; best = qq; }
        }
        const uint16_t x = so[l * 8 + best];
        so[l * 8 + best] = so[l * 8 + q];
        so[l * 8 + q] = x;
        ++cnt[x & 15];
      }
    }
  int steps = 0;
  while ((1 << steps) < gmax) ++steps;
  T.shdr[t] = (uint32_t)rounds | (uint32_t)steps << 8;
}

// G8 incidence groups: per tile node its (bank-scheduled) incidence list as contribution
// offsets w = a D kCbStride + el, padded with kTile (a zero column) to a multiple of 8;
// ptr8[r] = the node's first group.
__device__ int g8_entries(const uint16_t *ptr, int U) {
  int n8 = 0;
  for (int r = 0; r < U; ++r) n8 += (ptr[r + 1] - ptr[r] + 7) & ~7;
  return n8;
}

__global__ void k_g8_count(TileSet T, int *max_entries) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T.n_tiles) return;
  atomicMax(max_entries, g8_entries(T.ptr + t * (T.maxe + 1), T.U[t]));
}

template <int D>
__global__ void k_g8_fill(TileSet T, int me8, uint16_t *inc8, uint16_t *ptr8) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T.n_tiles) return;
  const int U = T.U[t];
  const uint16_t *ptr = T.ptr + t * (T.maxe + 1);
  const uint16_t *inc = T.inc + t * T.maxe;
  uint16_t *o = inc8 + t * (int64_t)me8;
  uint16_t *pg = ptr8 + t * (int64_t)(T.um + 1);
  int w = 0;
  for (int r = 0; r < U; ++r) {
    pg[r] = (uint16_t)(w / 8);
    const int lo = ptr[r], n = ptr[r + 1] - lo, n8 = (n + 7) & ~7;
    for (int q = 0; q < n8; ++q) {
      const int e = q < n ? inc[lo + q] : -1;
      o[w + q] = e < 0 ? (uint16_t)kTile : (uint16_t)((e & 3) * D * kCbStrideG8 + (e >> 2));
    }
    w += n8;
  }
  for (int r = U; r <= T.um; ++r) pg[r] = (uint16_t)(w / 8);
  for (; w < me8; ++w) o[w] = (uint16_t)kTile;
}

fem_status pack_tile_meta(Problem *p, cudaStream_t s) {
  TileSet &T = p->tiles;
  if (FEM_P2_BAL) {
    int *d_max = nullptr, h_max = 0;
    FEM_CUDA(cudaMalloc(&d_max, sizeof(int)));
    FEM_CUDA(cudaMemsetAsync(d_max, 0, sizeof(int), s));
    const unsigned g = (unsigned)((T.n_tiles + 127) / 128);
    k_sched_count<<<g, 128, 0, s>>>(T, d_max);
    FEM_CUDA(cudaMemcpyAsync(&h_max, d_max, sizeof(int), cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_max);
    T.sched_rounds = std::max(1, (h_max + kTile - 1) / kTile);
    const int64_t cap = (int64_t)T.sched_rounds * kTile;
    FEM_CUDA(cudaMalloc(&T.soff, sizeof(uint16_t) * 8 * cap * T.n_tiles));
    FEM_CUDA(cudaMalloc(&T.smeta, sizeof(uint32_t) * cap * T.n_tiles));
    FEM_CUDA(cudaMalloc(&T.shdr, sizeof(uint32_t) * T.n_tiles));
    if (p->dim == 3) k_build_sched<3><<<g, 128, 0, s>>>(T, T.sched_rounds);
    else k_build_sched<2><<<g, 128, 0, s>>>(T, T.sched_rounds);
    FEM_LAUNCH_CHECK("phase-2 schedule");
  }
  const bool lsplit = FEM_P2_LSPLIT > 0 && p->dim == 3 && !FEM_P2_BAL && !FEM_P2_G8 && !FEM_P2_NM && !FEM_P2_PAIR &&
                      !getenv("FEM_P2_LSPLIT_OFF");
  if (FEM_P2_SORT && !FEM_P2_BAL && !FEM_P2_G8 && !FEM_P2_NM && !FEM_P2_PAIR && !lsplit) {
    FEM_CUDA(cudaMalloc(&T.p2perm, sizeof(uint16_t) * (size_t)T.n_tiles * T.maxe));
    k_p2_perm<<<(unsigned)((T.n_tiles + 127) / 128), 128, 0, s>>>(T);
    FEM_LAUNCH_CHECK("phase-2 node order");
  }
  if (FEM_TILE_SCHED && !FEM_P2_BAL) {
    k_sched_inc<<<(unsigned)T.n_tiles, 8, 0, s>>>(T);
    FEM_LAUNCH_CHECK("tile incidence scheduling");
  }
  T.um = round_up(T.max_U > 0 ? T.max_U : 1, 8);
  T.pcap = T.um;
  if (lsplit) {  // tasks: <= 2 U per tile
    FEM_CUDA(cudaMalloc(&T.p2perm, sizeof(uint16_t) * (size_t)T.n_tiles * T.maxe));
    FEM_CUDA(cudaMalloc(&T.p2n, sizeof(int32_t) * (size_t)T.n_tiles));
    k_p2_tasks<<<(unsigned)((T.n_tiles + 127) / 128), 128, 0, s>>>(T, FEM_P2_LSPLIT);
    FEM_LAUNCH_CHECK("phase-2 tasks");
    T.pcap = std::min(2 * T.um, T.maxe);
  }
  if (FEM_P2_G8) {  // padded incidence groups (k_g8_fill), staged for k_pack_meta
    int *d_max = nullptr, h_max = 0;
    FEM_CUDA(cudaMalloc(&d_max, sizeof(int)));
    FEM_CUDA(cudaMemsetAsync(d_max, 0, sizeof(int), s));
    const unsigned g = (unsigned)((T.n_tiles + 127) / 128);
    k_g8_count<<<g, 128, 0, s>>>(T, d_max);
    FEM_CUDA(cudaMemcpyAsync(&h_max, d_max, sizeof(int), cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_max);
    T.me8 = round_up(std::max(h_max, 8), 8);
    FEM_CUDA(cudaMalloc(&T.inc8, sizeof(uint16_t) * (size_t)T.me8 * T.n_tiles));
    FEM_CUDA(cudaMalloc(&T.ptr8, sizeof(uint16_t) * (size_t)(T.um + 1) * T.n_tiles));
    if (p->dim == 3) k_g8_fill<3><<<g, 128, 0, s>>>(T, T.me8, T.inc8, T.ptr8);
    else k_g8_fill<2><<<g, 128, 0, s>>>(T, T.me8, T.inc8, T.ptr8);
    FEM_LAUNCH_CHECK("phase-2 incidence groups");
  }
  T.off_nodes = 16;
  T.off_lconn = T.off_nodes + 4 * T.um;
  if (FEM_P2_BAL) {
    const int cap = T.sched_rounds * kTile;
    T.off_soff = T.off_lconn + 8 * kTile;
    T.off_smeta = T.off_soff + 16 * cap;
    T.off_int = T.off_smeta + 4 * cap;
    T.off_ptr = T.off_inc = -1;
  } else if (FEM_P2_G8) {
    T.off_ptr = T.off_lconn + 8 * kTile;
    T.off_inc = T.off_ptr + round_up(2 * (T.um + 1), 16);
    T.off_int = T.off_inc + round_up(2 * T.me8, 16);
  } else {
    T.off_ptr = T.off_lconn + 8 * kTile;
    T.off_inc = T.off_ptr + round_up(2 * (T.um + 1), 16);
    T.off_int = T.off_inc + 8 * kTile;
  }
  T.off_bc = T.off_int + round_up(T.um, 16);
  T.off_ph = T.off_bc + round_up(T.um, 16);
  T.off_perm = round_up(T.off_ph + (T.phase ? kTile : 0), 16);
  T.mb = round_up(T.off_perm + (T.p2perm ? 2 * T.pcap : 0), 16);
  FEM_CUDA(cudaMalloc(&T.meta, (size_t)T.mb * T.n_tiles));
  if (p->dim == 2) k_pack_meta<2><<<(unsigned)T.n_tiles, 256, 0, s>>>(T, p->node_bc, p->n_elems);
  else k_pack_meta<3><<<(unsigned)T.n_tiles, 256, 0, s>>>(T, p->node_bc, p->n_elems);
  FEM_LAUNCH_CHECK("pack tile meta");
  if (FEM_HVP_G8 && !FEM_P2_G8 && !FEM_P2_BAL && !FEM_P2_NM && !FEM_P2_PAIR && !FEM_WS && !T.meta_g8) {
    // HVP metadata with the incidences in padded groups of 8 (k_g8_fill), packed by
    // k_pack_meta from a copy of the tile set carrying the G8 layout
    int *d_max = nullptr, h_max = 0;
    FEM_CUDA(cudaMalloc(&d_max, sizeof(int)));
    FEM_CUDA(cudaMemsetAsync(d_max, 0, sizeof(int), s));
    const unsigned g = (unsigned)((T.n_tiles + 127) / 128);
    k_g8_count<<<g, 128, 0, s>>>(T, d_max);
    FEM_CUDA(cudaMemcpyAsync(&h_max, d_max, sizeof(int), cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaStreamSynchronize(s));
    cudaFree(d_max);
    TileSet T2 = T;
    T2.me8 = round_up(std::max(h_max, 8), 8);
    FEM_CUDA(cudaMalloc(&T2.inc8, sizeof(uint16_t) * (size_t)T2.me8 * T.n_tiles));
    FEM_CUDA(cudaMalloc(&T2.ptr8, sizeof(uint16_t) * (size_t)(T.um + 1) * T.n_tiles));
    if (p->dim == 3) k_g8_fill<3><<<g, 128, 0, s>>>(T2, T2.me8, T2.inc8, T2.ptr8);
    else k_g8_fill<2><<<g, 128, 0, s>>>(T2, T2.me8, T2.inc8, T2.ptr8);
    FEM_LAUNCH_CHECK("phase-2 incidence groups (HVP)");
    T2.p2perm = nullptr;
    T2.p2n = nullptr;
    T2.pcap = 0;
    T2.shdr = nullptr;
    T2.off_inc = T.off_ptr + round_up(2 * (T.um + 1), 16);
    T2.off_int = T2.off_inc + round_up(2 * T2.me8, 16);
    T2.off_bc = T2.off_int + round_up(T.um, 16);
    T2.off_ph = T2.off_bc + round_up(T.um, 16);
    T2.off_perm = round_up(T2.off_ph + (T.phase ? kTile : 0), 16);
    T2.mb = round_up(T2.off_perm, 16);
    FEM_CUDA(cudaMalloc(&T2.meta, (size_t)T2.mb * T.n_tiles));
    if (p->dim == 2) k_pack_meta<2><<<(unsigned)T.n_tiles, 256, 0, s>>>(T2, p->node_bc, p->n_elems);
    else k_pack_meta<3><<<(unsigned)T.n_tiles, 256, 0, s>>>(T2, p->node_bc, p->n_elems);
    FEM_LAUNCH_CHECK("pack tile meta (HVP)");
    FEM_CUDA(cudaStreamSynchronize(s));
    cudaFree(T2.inc8);
    cudaFree(T2.ptr8);
    T.meta_g8 = T2.meta;
    T.mb_g8 = T2.mb;
    T.off_inc_g8 = T2.off_inc;
    T.off_int_g8 = T2.off_int;
    T.off_bc_g8 = T2.off_bc;
    T.off_ph_g8 = T2.off_ph;
    T.off_perm_g8 = T2.off_perm;
  }
  if (T.inc8) {
    FEM_CUDA(cudaStreamSynchronize(s));
    cudaFree(T.inc8); cudaFree(T.ptr8);
    T.inc8 = nullptr; T.ptr8 = nullptr;
  }
  if (FEM_P2_BAL) {  // packed into the metadata blocks: the staging copies are not needed
    FEM_CUDA(cudaStreamSynchronize(s));
    cudaFree(T.soff); cudaFree(T.smeta); cudaFree(T.shdr);
    T.soff = nullptr; T.smeta = nullptr; T.shdr = nullptr;
  }
  return FEM_OK;
}

// ------------------------------------------------------------------ pipelined tile kernels
// Persistent CTAs walk the tiles t = blockIdx.x, +gridDim.x, ...  While tile k is computed,
// cp.async copies of tile k+1's nodal data (8-byte gathers of coordinates, u, v) and tile
// k+2's metadata block (16-byte copies) are in flight: meta is triple-, node data
// double-buffered in shared memory, so HBM/L2 latency overlaps the FP64 element math.
// cp.async / mbarrier / TMA bulk-copy helpers: pipe.cuh


// CTAs per SM the register budget targets (A/B on cfg 3, profiles/): the NH HVP is the
// register-heaviest and runs fastest spill-free at 2; energy at 4; residual at 3.
// (stated for 256-thread CTAs; smaller tiles scale the CTA count so warps/SM stay equal)
// 2D elements need far fewer registers (46-68): more CTAs per SM.  A/B at the cfg 2 size
// (10M DOFs, CTAs/SM 2/3/4/5): HVP 0.340/0.303/0.344/0.344 ms, residual (3 by default)
// 0.266/0.266/0.255/0.251 ms, energy (4 by default) 0.166/0.172/0.170/0.163 ms.
__host__ __device__ constexpr int pipe_minb2d(int op, int mat) {
  return op == OP_RESIDUAL_S || op == OP_HVP_S ? 3 : op == OP_ENERGY || op == OP_RESIDUAL || op == OP_LIN ? 5
         : (mat == FEM_NEO_HOOKEAN ? 3 : 4);
}
#ifndef FEM_HVPR_MINB
#define FEM_HVPR_MINB 2
#endif
#ifndef FEM_RESR_MINB
#define FEM_RESR_MINB 3
#endif
__host__ __device__ constexpr int pipe_minb(int op, int mat, int dim = 3) {
#ifdef FEM_HVPR_CTAS
  if (op == OP_HVP_R && dim == 3) return FEM_HVPR_CTAS;
#endif
  return op == OP_HVP_R ? (256 / kTile) * (dim == 2 ? 3 : FEM_HVPR_MINB)
         : op == OP_RESIDUAL_R ? (256 / kTile) * (dim == 2 ? 5 : FEM_RESR_MINB) :
         (256 / kTile) *
         (dim == 2 ? (FEM_PIPE_MINB2D > 0 ? FEM_PIPE_MINB2D : pipe_minb2d(op, mat))
          : FEM_PIPE_MINB > 0 ? FEM_PIPE_MINB
                            : (op == OP_RESIDUAL_S || op == OP_HVP_S) ? 2
                            : (op == OP_ENERGY ? 4 : (op == OP_RESIDUAL ? FEM_RES_MINB : op == OP_LIN ? 3
                                : (op == OP_HVP_LIN ? 3 : (mat == FEM_NEO_HOOKEAN ? FEM_HVP_MINB : 3)))));
}

struct PipeArgs {
  const uint8_t *meta;
  int64_t n_tiles, E;
  int mb, um, off_nodes, off_lconn, off_ptr, off_inc, off_int, off_bc, off_ph, off_soff, off_smeta, off_perm;
  bool has_phase, has_perm;
  const int64_t *slot_off;
  const double *coords, *u, *v;
  double lam, mu;
  const double *lam_tab, *mu_tab;
  double *out, *slots, *partials;
  const int32_t *list;  // tile ids to process (null: tiles 0 .. n_tiles-1)
  double *lin;        // linearization cache [lin_words][lin_stride] (OP_LIN writes, OP_HVP_LIN reads)
  const double *geom; // OP_*_S: per-tile geometry blocks [n_tiles][D*D+1][kTile]
  const double *refm; // OP_*_R: per-tile reference metric blocks [n_tiles][refm_words(D)][kTile]
  int64_t lin_stride;
  int *err;
};

template <int OP>
constexpr bool op_streams() { return OP == OP_RESIDUAL_S || OP == OP_HVP_S; }
template <int OP>  // the operation an OP_*_S / OP_*_R variant computes
constexpr int base_op() {
  return (OP == OP_RESIDUAL_S || OP == OP_RESIDUAL_R) ? OP_RESIDUAL
         : (OP == OP_HVP_S || OP == OP_HVP_R) ? OP_HVP : OP;
}
template <int OP>
constexpr bool op_is_hvp() { return OP == OP_HVP || OP == OP_HVP_LIN || OP == OP_HVP_S || OP == OP_HVP_R; }
template <int OP>
constexpr bool op_refm() { return OP == OP_RESIDUAL_R || OP == OP_HVP_R; }
// reference metric per element (OP_*_R): mu vol G_a.G_b for 1 <= a <= b <= D (row-major upper
// triangle) and 1 / det J(x)
__host__ __device__ constexpr int refm_words(int D) { return D * (D + 1) / 2 + 1; }
__host__ __device__ constexpr int sym_idx(int a, int b, int D) {  // upper-triangle position
  return a <= b ? a * D - a * (a - 1) / 2 + (b - a) : b * D - b * (b - 1) / 2 + (a - b);
}
template <int OP>
constexpr bool op_has_p2() { return !FEM_P1_RED && (base_op<OP>() == OP_RESIDUAL || op_is_hvp<OP>()); }
template <int OP>
constexpr bool op_scatters() { return base_op<OP>() == OP_RESIDUAL || op_is_hvp<OP>(); }
// the G8 node sums: every phase-2 op with FEM_P2_G8, else the HVP ops with FEM_HVP_G8 (their
// metadata comes from TileSet::meta_g8)
template <int OP>
constexpr bool op_g8() {
  return FEM_P2_G8 ? op_has_p2<OP>()
                   : (FEM_HVP_G8 && !FEM_P2_BAL && !FEM_P2_NM && !FEM_P2_PAIR && !FEM_WS &&
                      OP == OP_HVP);  // the linearized HVP measured slower with G8 (0.961 vs 0.737 ms)
}
template <int OP>
constexpr int cb_stride() { return op_g8<OP>() ? kCbStrideG8 : kTile; }
template <int OP, int MAT>
constexpr bool op_needs_u() {
  return OP == OP_ENERGY || base_op<OP>() == OP_RESIDUAL || OP == OP_LIN ||
         (base_op<OP>() == OP_HVP && MAT == FEM_NEO_HOOKEAN);
}
constexpr int geom_words(int D) { return D * D + 1; }
template <int OP, int MAT>  // the coordinates are staged unless the geometry comes from a stream / cache
constexpr bool op_needs_x() { return !op_streams<OP>() && !(OP == OP_HVP_LIN && MAT == FEM_NEO_HOOKEAN); }
// fem_linearize cache per element (NH, deformed-configuration metric form of the HVP):
// cs_a (D x D), s1 = c1 / (d! J det J(x+u)), s2 = lam / (d! J det J(x+u)), Ms (D(D+1)/2,
// symmetric: mu (c_a . c_b) / (d! det J(x)))
__host__ __device__ constexpr int lin_words(int D) { return D * D + 2 + D * (D + 1) / 2; }

template <int D, int MAT, int OP_, bool MASK>
__device__ __forceinline__ void tile_phase1(const PipeArgs &A, const unsigned char *m,
                                            const double *xs, const double *us, const double *vs,
                                            int64_t t, int tid, double *cb, double &eacc,
                                            const double *gs = nullptr) {
  // OP_*_S: the same operation with c_a, det J read from the streamed geometry block gs
  constexpr int OP = base_op<OP_>();
  constexpr bool STREAM = op_streams<OP_>();
  // OP_*_R: the reference metric mu vol G_a.G_b and 1/det J come from the per-element cache,
  // so the reference cofactors c_a are never formed (only the deformed geometry at x + u)
  constexpr bool REFM = op_refm<OP_>();
  constexpr int RW = refm_words(D);
  constexpr int NEN = D + 1;
  constexpr bool NEED_U = op_needs_u<OP, MAT>();
  // NH HVP in the deformed configuration (FEM_HVP_SPATIAL): see the HVP branch below; the
  // streamed form has no coordinates and runs the material form (F = I + H, F^-T, ln J)
  constexpr bool SPATIAL = FEM_HVP_SPATIAL && OP == OP_HVP && MAT == FEM_NEO_HOOKEAN && !STREAM;
  // NH residual with F^-T G_a from the same deformed geometry (FEM_RES_SPATIAL)
  constexpr bool SPATIAL_R = FEM_RES_SPATIAL && OP == OP_RESIDUAL && MAT == FEM_NEO_HOOKEAN && !STREAM;
  // linearization (OP_LIN) caches the deformed-configuration metric form; the cached HVP
  // (OP_HVP_LIN) then needs no geometry at all
  constexpr bool LIN_S = OP == OP_LIN && MAT == FEM_NEO_HOOKEAN;
  constexpr bool NO_GEOM = OP == OP_HVP_LIN && MAT == FEM_NEO_HOOKEAN;
  const int64_t e = t * kTile + tid;
  if (e < A.E) {
    const ushort4 lc4 = reinterpret_cast<const ushort4 *>(m + A.off_lconn)[tid];
    const int lc[4] = {lc4.x, lc4.y, lc4.z, lc4.w};
    double rm[RW];
    if constexpr (REFM) {  // coalesced over the tile (SoA), L2-prefetched one tile ahead
      const double *R = A.refm + t * (RW * kTile) + tid;
#pragma unroll
      for (int w = 0; w < RW; ++w) rm[w] = __ldg(R + w * kTile);
    }
    double x[NEN][D], c[D][D], det;
    if constexpr (NO_GEOM) {
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int j = 0; j < D; ++j) c[a][j] = 0.0;
      det = 1.0;
    } else if constexpr (STREAM) {  // Alg. 1's gathered geometry: c_a = det G_a, det J
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int j = 0; j < D; ++j) c[a][j] = gs[(a * D + j) * kTile + tid];
      det = gs[D * D * kTile + tid];
    } else {
#pragma unroll
      for (int a = 0; a < NEN; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) x[a][i] = xs[lc[a] * D + i];
      if constexpr (REFM) {
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int j = 0; j < D; ++j) c[a][j] = 0.0;
        det = 1.0;
      } else {
        det = cof_gradients<D>(x, c);
      }
    }
    const double id = REFM ? rm[RW - 1] : fem_rcp(det);
    constexpr double inv_fact = (D == 3) ? 1.0 / 6.0 : 0.5;  // vol = det / d!
    double lam = A.lam, mu = A.mu;
    if (A.has_phase) {
      const int ph = m[A.off_ph + tid];
      lam = A.lam_tab[ph];
      mu = A.mu_tab[ph];
    }
    double H[D][D];
    double cs[D][D], dets = 1.0;  // SPATIAL: cofactor gradients and det J at x + u
    double xd[NEN][D];            // deformed edge vectors (SPATIAL forms)
    if constexpr (NEED_U) {
      double u[NEN][D];
#pragma unroll
      for (int a = 0; a < NEN; ++a)
#pragma unroll
        for (int i = 0; i < D; ++i) u[a][i] = us[lc[a] * D + i];
      if constexpr (SPATIAL_R && !REFM) grad_hat<D>(u, c, H);  // Hh = det H (scaled where used)
      if constexpr (SPATIAL || SPATIAL_R || LIN_S) {
        deformed_edges<D>(x, u, xd);
        dets = cof_gradients<D>(xd, cs);
      } else {
        grad_hat<D>(u, c, H);
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int j = 0; j < D; ++j) H[i][j] *= id;
      }
    }
    double f[NEN][D];  // SPATIAL: the nodal vectors, formed in the HVP branch
    bool ok = true;
    double S[D][D];
    if constexpr (OP == OP_ENERGY) {
      const double vol = det * inv_fact;
      if constexpr (MAT == FEM_LINEAR_ELASTIC) {
        eacc += vol * le_psi<D>(H, lam, mu);
      } else {
        NHState<D> s;
        ok = nh_state<D>(H, s);
        if (ok) eacc += vol * nh_psi<D>(H, s, lam, mu);
      }
    } else if constexpr (OP == OP_RESIDUAL) {
      // vol P G_a = (P / d!) c_a; P linear in (lambda, mu).  With partials (fem_energy_residual)
      // the element energy vol psi(H) is accumulated in the same pass (value and gradient).
      const double ls = lam * inv_fact, ms = mu * inv_fact;
      const double vol = det * inv_fact;
      if constexpr (MAT == FEM_LINEAR_ELASTIC) {
        le_stress<D>(H, ls, ms, S);
        if (A.partials) eacc += vol * le_psi<D>(H, lam, mu);
      } else if constexpr (SPATIAL_R) {
        // P = mu (F - F^-T) + lam ln J F^-T with F c_a = c_a + Hh c_a / det and
        // F^-T c_a = det g_a = cs_a / J (g_a: gradients at x + u, J = det J(x+u) / det J(x)):
        //   vol P G_a = (1/d!) [mu c_a + (mu/det) Hh c_a + ((lam ln J - mu) / J) cs_a], a >= 1
        const double Jr = dets * id;
        ok = Jr > 0.0;
        const double lnJ = fem_log(Jr);
        const double kc = (lam * lnJ - mu) * fem_rcp(Jr) * inv_fact, kh = ms * id;
        if constexpr (REFM) {
          // mu vol F G_a = mu vol sum_b xd_b (G_b.G_a) (F = sum_b xd_b (x) G_b over the deformed
          // edges): vol P G_a = sum_b Ms_ab xd_b + kc cs_a, a >= 1 — the same terms as below
          // (sum_b Ms_ab (x_b - x_0) = mu c_a / d!), from the cached metric Ms
#pragma unroll
          for (int i = 0; i < D; ++i) {
            double s0 = 0.0;
#pragma unroll
            for (int a = 0; a < D; ++a) {
              double fa = kc * cs[a][i];
#pragma unroll
              for (int b = 0; b < D; ++b) fa = fma(rm[sym_idx(a, b, D)], xd[b + 1][i], fa);
              f[a + 1][i] = fa;
              s0 += fa;
            }
            f[0][i] = -s0;
          }
        } else {
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double s0 = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            double p = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) p = fma(H[i][j], c[a][j], p);
            const double fa = fma(ms, c[a][i], fma(kh, p, kc * cs[a][i]));
            f[a + 1][i] = fa;
            s0 += fa;
          }
          f[0][i] = -s0;
        }
        }
        if (!REFM && A.partials && ok) {  // psi from H = Hh / det: F:F - d = 2 tr H + H:H
          double th = 0.0;
#pragma unroll
          for (int i = 0; i < D; ++i) {
            th += 2.0 * (H[i][i] * id);
#pragma unroll
            for (int j = 0; j < D; ++j) th = fma(H[i][j] * id, H[i][j] * id, th);
          }
          eacc += vol * (0.5 * mu * (th - 2.0 * lnJ) + 0.5 * lam * lnJ * lnJ);
        }
      } else {
        NHState<D> s;
        ok = nh_state<D>(H, s);
        if (ok) {
          nh_stress<D>(s, ls, ms, S);
          if (A.partials) eacc += vol * nh_psi<D>(H, s, lam, mu);
        }
      }
    } else if constexpr (OP == OP_LIN) {
      if constexpr (MAT == FEM_NEO_HOOKEAN) {  // the metric-form tangent at this state (SoA)
        const double Jr = dets * id;
        ok = Jr > 0.0;
        const double scur = inv_fact * fem_rcp(Jr * dets);
        const double c1 = mu - lam * fem_log(Jr);
        const double sr = mu * id * inv_fact;
        double *L = A.lin + e;
        const int64_t st = A.lin_stride;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int j = 0; j < D; ++j) L[(a * D + j) * st] = ok ? cs[a][j] : 0.0;
        L[(D * D) * st] = ok ? scur * c1 : 0.0;
        L[(D * D + 1) * st] = ok ? scur * lam : 0.0;
        int q = D * D + 2;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = a; b < D; ++b) {
            double t = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) t = fma(c[a][j], c[b][j], t);
            L[(q++) * st] = ok ? sr * t : 0.0;
          }
      }
    } else if constexpr (NO_GEOM) {
      // cached HVP (FEM_LINEARIZED): the HVP's metric form with cs_a, s1 = k1 / c1... read
      // from the linearization — per element lin_words(D) loads instead of the geometry of
      // x and x + u, the log and the reciprocals
      const double *L = A.lin + e;
      const int64_t st = A.lin_stride;
      double csl[D][D], Ms[D][D];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int j = 0; j < D; ++j) csl[a][j] = __ldg(L + (a * D + j) * st);
      const double s1 = __ldg(L + (D * D) * st), s2 = __ldg(L + (D * D + 1) * st);
      {
        int q = D * D + 2;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = a; b < D; ++b) Ms[a][b] = Ms[b][a] = __ldg(L + (q++) * st);
      }
      double dv[D][D];
      {
        double v0[D];
        const unsigned bc0 = MASK ? m[A.off_bc + lc[0]] : 0u;
#pragma unroll
        for (int i = 0; i < D; ++i) v0[i] = (bc0 & (1u << i)) ? 0.0 : vs[lc[0] * D + i];
#pragma unroll
        for (int b = 0; b < D; ++b) {
          const unsigned bc = MASK ? m[A.off_bc + lc[b + 1]] : 0u;
#pragma unroll
          for (int i = 0; i < D; ++i)
            dv[b][i] = ((bc & (1u << i)) ? 0.0 : vs[lc[b + 1] * D + i]) - v0[i];
        }
      }
      double Dm[D][D], tr = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < D; ++j) t = fma(dv[b][j], csl[a][j], t);
          Dm[a][b] = t;
          if (a == b) tr += t;
        }
      const double k2 = s2 * tr;
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) Dm[a][b] = (a == b) ? fma(s1, Dm[a][b], k2) : s1 * Dm[a][b];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s0 = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          double fa = 0.0;
#pragma unroll
          for (int b = 0; b < D; ++b) fa = fma(Ms[a][b], dv[b][i], fma(Dm[a][b], csl[b][i], fa));
          f[a + 1][i] = fa;
          s0 += fa;
        }
        f[0][i] = -s0;
      }
    } else if constexpr (SPATIAL && FEM_HVP_MD) {
      // Deformed-configuration HVP (reading R9) in metric form.  With dv_b = v_b - v_0,
      // c_a the cofactor rows at x, cs_a those at x + u (g_a = cs_a / det J(x+u)):
      //   vol dP G_a = sr sum_b M_ab dv_b + sum_b (k1 D_ab + k2 delta_ab) cs_b,  a >= 1,
      //   M_ab = c_a . c_b,  D_ab = dv_b . cs_a,  tr A det J(x+u) = sum_b D_bb,
      //   sr = mu / (d! det), k1 = c1 s, k2 = lam tr(D) s, s = 1 / (d! J det J(x+u)),
      //   c1 = mu - lam ln J, J = det J(x+u) / det J(x); node 0 = minus the sum.
      // (the same terms as the dH / Ah form below: (dH c_a) = sum_b M_ab dv_b and
      // (Ah^T cs_a) = sum_b D_ab cs_b; 3x3 metrics replace two 3x3x3 products)
      double dv[D][D];
      {
        double v0[D];
        const unsigned bc0 = MASK ? m[A.off_bc + lc[0]] : 0u;
#pragma unroll
        for (int i = 0; i < D; ++i) v0[i] = (bc0 & (1u << i)) ? 0.0 : vs[lc[0] * D + i];
#pragma unroll
        for (int b = 0; b < D; ++b) {
          const unsigned bc = MASK ? m[A.off_bc + lc[b + 1]] : 0u;
#pragma unroll
          for (int i = 0; i < D; ++i)
            dv[b][i] = ((bc & (1u << i)) ? 0.0 : vs[lc[b + 1] * D + i]) - v0[i];
        }
      }
      const double Jr = dets * id;
      ok = Jr > 0.0;
      const double c1 = mu - lam * fem_log(Jr);
      const double sr = mu * id * inv_fact, scur = inv_fact * fem_rcp(Jr * dets);
      double Dm[D][D], tr = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double t = 0.0;
#pragma unroll
          for (int j = 0; j < D; ++j) t = fma(dv[b][j], cs[a][j], t);
          Dm[a][b] = t;
          if (a == b) tr += t;
        }
      const double k1 = scur * c1, k2 = scur * lam * tr;
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) Dm[a][b] = (a == b) ? fma(k1, Dm[a][b], k2) : k1 * Dm[a][b];
      double Ms[D][D];
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = a; b < D; ++b) {
          if constexpr (REFM) {
            Ms[a][b] = Ms[b][a] = rm[sym_idx(a, b, D)];
          } else {
            double t = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) t = fma(c[a][j], c[b][j], t);
            Ms[a][b] = Ms[b][a] = sr * t;
          }
        }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s0 = 0.0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          double fa = 0.0;
#pragma unroll
          for (int b = 0; b < D; ++b) fa = fma(Ms[a][b], dv[b][i], fma(Dm[a][b], cs[b][i], fa));
          f[a + 1][i] = fa;
          s0 += fa;
        }
        f[0][i] = -s0;
      }
    } else {
      // dH = dHh / det; vol dP(dH) G_a = dP(dHh) c_a * (1 / (det d!)): fold into (lambda, mu)
      double v[NEN][D], dH[D][D];
#pragma unroll
      for (int a = 0; a < NEN; ++a) {
        const unsigned bc = MASK ? m[A.off_bc + lc[a]] : 0u;
#pragma unroll
        for (int i = 0; i < D; ++i) v[a][i] = (bc & (1u << i)) ? 0.0 : vs[lc[a] * D + i];
      }
      grad_hat<D>(v, c, dH);
      const double sc = id * inv_fact;
      const double ls = lam * sc, ms = mu * sc;
      if constexpr (SPATIAL) {
        // g_b = F^-T G_b = cs_b / det J(x+u) are the deformed-configuration gradients, so
        // A = dH F^-1 = sum_b v_b (x) g_b = Ah / det J(x+u) (Ah = grad_hat(v, cs)),
        // F^-T dH^T F^-T G_a = A^T g_a and F^-T : dH = tr A.  With J = det J(x+u) / det J(x):
        //   vol dP G_a = mu/(d! det) dHh c_a + 1/(d! J det J(x+u)) (c1 Ah^T cs_a + lam tr(Ah) cs_a)
        // for a >= 1 (c1 = mu - lam ln J), and minus their sum for a = 0.  F, F^-1 and H are
        // never formed; the two geometry chains (x and x + u) are independent.
        double Ah[D][D];
        grad_hat<D>(v, cs, Ah);
        const double Jr = dets * id;
        ok = Jr > 0.0;
        const double c1 = mu - lam * fem_log(Jr);
        const double sr = mu * sc, scur = inv_fact * fem_rcp(Jr * dets);
        double tr = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) tr += Ah[k][k];
        const double ltr = lam * tr;
#pragma unroll
        for (int i = 0; i < D; ++i) {
          double s0 = 0.0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            double p = 0.0, q = ltr * cs[a][i], w = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) {
              p = fma(dH[i][j], c[a][j], p);
              w = fma(Ah[j][i], cs[a][j], w);
            }
            const double fa = fma(sr, p, scur * fma(c1, w, q));
            f[a + 1][i] = fa;
            s0 += fa;
          }
          f[0][i] = -s0;
        }
      } else if constexpr (MAT == FEM_LINEAR_ELASTIC) {
        le_stress<D>(dH, ls, ms, S);
      } else {
        NHState<D> s;
        ok = nh_state<D>(H, s);
        if (ok) nh_dstress<D>(s, ls, ms, dH, S);
      }
    }
    if (!ok) atomicOr(A.err, ERRW_INVERTED);
    if constexpr (op_scatters<OP>()) {
      if constexpr (!SPATIAL && !SPATIAL_R && !NO_GEOM) nodal_from_c<D>(S, c, f);
      if constexpr (FEM_P1_RED) {
        const int32_t *nodes = reinterpret_cast<const int32_t *>(m + A.off_nodes);
#pragma unroll
        for (int a = 0; a < NEN; ++a)
#pragma unroll
          for (int i = 0; i < D; ++i) atomicAdd(A.out + (int64_t)nodes[lc[a]] * D + i, f[a][i]);
      } else {
#pragma unroll
        for (int a = 0; a < NEN; ++a)
#pragma unroll
          for (int i = 0; i < D; ++i) {
            if constexpr (FEM_P2_NM) {  // node-major: at the incidence's list position
              const int q = reinterpret_cast<const uint16_t *>(m + A.off_inc)[tid * 4 + a];
              cb[q * D + i] = ok ? f[a][i] : 0.0;
            } else {
              cb[(a * D + i) * cb_stride<OP_>() + tid] = ok ? f[a][i] : 0.0;
            }
          }
      }
    }
  }
}

// Phase 2: fixed-order per-tile-node sums of the contributions, stored (interior nodes),
// RED (tile-boundary nodes) or written to the node's slot (DET).
// Scatter mode SC of the tile-boundary nodes: 0 RED (default), 1 the node's slot (DET),
// 2 plain read-add-write (tile-colored passes: tiles of one color share no node).
template <int D, int SC>
__device__ __forceinline__ void node_write(const PipeArgs &A, const unsigned char *m, int r,
                                           int64_t t, const double (&sacc)[D]) {
  if constexpr (SC == 1) {
    double *slot = A.slots + (A.slot_off[t] + r) * D;
#pragma unroll
    for (int cc = 0; cc < D; ++cc) slot[cc] = sacc[cc];
  } else {
    const int32_t *nodes = reinterpret_cast<const int32_t *>(m + A.off_nodes);
    const int64_t g = (int64_t)nodes[r] * D;
    if (m[A.off_int + r]) {
#pragma unroll
      for (int cc = 0; cc < D; ++cc) A.out[g + cc] = sacc[cc];
    } else if constexpr (SC == 2) {
#pragma unroll
      for (int cc = 0; cc < D; ++cc) A.out[g + cc] += sacc[cc];
    } else {
#pragma unroll
      for (int cc = 0; cc < D; ++cc) atomicAdd(A.out + g + cc, sacc[cc]);
    }
  }
}

// One thread per tile node; the node's entries come in groups of 8 contribution offsets
// (16-byte loads), pad entries point at the zero columns; two interleaved partial sums.
template <int D, int OP, int SC>
__device__ __forceinline__ void tile_phase2_g8(const PipeArgs &A, const unsigned char *m, int U,
                                            int64_t t, int tid, const double *cb) {
  const uint16_t *ptr = reinterpret_cast<const uint16_t *>(m + A.off_ptr);
  const uint4 *grp = reinterpret_cast<const uint4 *>(m + A.off_inc);
  for (int r = tid; r < U; r += kTile) {
    const int g0 = ptr[r], g1 = ptr[r + 1];
    double s0[D], s1[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) s0[cc] = s1[cc] = 0.0;
    for (int g = g0; g < g1; ++g) {
      const uint4 o4 = grp[g];
      const uint32_t ow[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const double *pq = cb + ((ow[q >> 1] >> ((q & 1) * 16)) & 0xffffu);
#pragma unroll
        for (int cc = 0; cc < D; ++cc) {
          if (q & 1) s1[cc] += pq[cc * kCbStrideG8];
          else s0[cc] += pq[cc * kCbStrideG8];
        }
      }
    }
    double sacc[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) sacc[cc] = s0[cc] + s1[cc];
    node_write<D, SC>(A, m, r, t, sacc);
  }
}
#if FEM_P2_BAL
// Balanced schedule (k_build_sched): every thread sums one task of <= 8 incidences of one
// node from precomputed offsets; the g lanes of a node combine by a shuffle tree.
template <int D, int OP, int SC>
__device__ __forceinline__ void tile_phase2(const PipeArgs &A, const unsigned char *m, int U,
                                            int64_t t, int tid, const double *cb,
                                            int /*nth: default variant only*/ = kTile) {
  const uint32_t hdr = reinterpret_cast<const uint32_t *>(m)[2];
  const int rounds = hdr & 0xff, steps = (hdr >> 8) & 0xff;
  const uint4 *so = reinterpret_cast<const uint4 *>(m + A.off_soff);
  const uint32_t *sm = reinterpret_cast<const uint32_t *>(m + A.off_smeta);
  for (int rd = 0; rd < rounds; ++rd) {   // uniform over the CTA (shuffles below)
    const int j = rd * kTile + tid;
    const uint32_t mt = sm[j];
    const uint4 o4 = so[j];
    const int n = (mt >> 11) & 15, pos = (mt >> 15) & 0xff, g = (mt >> 23) & 0xff;
    const uint32_t ow[4] = {o4.x, o4.y, o4.z, o4.w};
    double s0[D], s1[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) s0[cc] = s1[cc] = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < n) {
        const double *pq = cb + ((ow[q >> 1] >> ((q & 1) * 16)) & 0xffffu);
#pragma unroll
        for (int cc = 0; cc < D; ++cc) {
          if (q & 1) s1[cc] += pq[cc * kTile];
          else s0[cc] += pq[cc * kTile];
        }
      }
    }
    double sacc[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) sacc[cc] = s0[cc] + s1[cc];
    for (int st = 0; st < steps; ++st) {
      const int off = 1 << st;
      const bool take = (pos & (2 * off - 1)) == 0 && pos + off < g;
#pragma unroll
      for (int cc = 0; cc < D; ++cc) {
        const double x = __shfl_down_sync(0xffffffffu, sacc[cc], off);
        if (take) sacc[cc] += x;
      }
    }
    if (n > 0 && pos == 0) node_write<D, SC>(A, m, (int)(mt & 0x7ffu), t, sacc);
  }
}
#elif FEM_P2_NM
template <int D, int OP, int SC>
__device__ __forceinline__ void tile_phase2(const PipeArgs &A, const unsigned char *m, int U,
                                            int64_t t, int tid, const double *cb,
                                            int /*nth: default variant only*/ = kTile) {
  const uint16_t *ptr = reinterpret_cast<const uint16_t *>(m + A.off_ptr);
  for (int r = tid; r < U; r += kTile) {  // one thread per tile node: a contiguous run
    const int lo = ptr[r], hi = ptr[r + 1];
    double s0[D], s1[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) s0[cc] = s1[cc] = 0.0;
    int q = lo;
    for (; q + 3 < hi; q += 4) {
#pragma unroll
      for (int cc = 0; cc < D; ++cc) {
        s0[cc] += cb[q * D + cc];
        s1[cc] += cb[(q + 1) * D + cc];
        s0[cc] += cb[(q + 2) * D + cc];
        s1[cc] += cb[(q + 3) * D + cc];
      }
    }
    for (; q < hi; ++q)
#pragma unroll
      for (int cc = 0; cc < D; ++cc) s0[cc] += cb[q * D + cc];
    double sacc[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) sacc[cc] = s0[cc] + s1[cc];
    node_write<D, SC>(A, m, r, t, sacc);
  }
}
#elif FEM_P2_G8
template <int D, int OP, int SC>
__device__ __forceinline__ void tile_phase2(const PipeArgs &A, const unsigned char *m, int U,
                                            int64_t t, int tid, const double *cb,
                                            int /*nth: default variant only*/ = kTile) {
  tile_phase2_g8<D, OP, SC>(A, m, U, t, tid, cb);
}
#elif FEM_P2_PAIR
// Two lanes per tile node (lanes 2r, 2r+1 of the CTA): each sums half of the node's
// incidence list (two interleaved partial sums), the pair combines by one shuffle per
// component and the even lane writes.  Up to 128 nodes per pass, so all 8 warps share the
// node sums instead of ceil(U / 32) of them (the critical path before the next tile's barrier).
template <int D, int OP, int SC>
__device__ __forceinline__ void tile_phase2(const PipeArgs &A, const unsigned char *m, int U,
                                            int64_t t, int tid, const double *cb,
                                            int /*nth: default variant only*/ = kTile) {
  const uint16_t *ptr = reinterpret_cast<const uint16_t *>(m + A.off_ptr);
  const uint16_t *inc = reinterpret_cast<const uint16_t *>(m + A.off_inc);
  for (int base = 0; base < 2 * U; base += kTile) {  // uniform over the CTA (shuffles)
    const int r2 = base + tid, r = r2 >> 1, half = r2 & 1;
    double s0[D], s1[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) s0[cc] = s1[cc] = 0.0;
    if (r < U) {
      const int lo = ptr[r], hi = ptr[r + 1], mid = (lo + hi + 1) >> 1;
      int w = half ? mid : lo;
      const int e = half ? hi : mid;
      for (; w + 1 < e; w += 2) {
        const int p0 = inc[w], p1 = inc[w + 1];
#pragma unroll
        for (int cc = 0; cc < D; ++cc) {
          s0[cc] += cb[p0 + cc * kTile];
          s1[cc] += cb[p1 + cc * kTile];
        }
      }
      if (w < e) {
        const int pk = inc[w];
#pragma unroll
        for (int cc = 0; cc < D; ++cc) s0[cc] += cb[pk + cc * kTile];
      }
    }
    double sacc[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) {
      const double own = s0[cc] + s1[cc];
      const double oth = __shfl_xor_sync(0xffffffffu, own, 1);
      sacc[cc] = half ? oth + own : own + oth;   // (first half) + (second half) on both lanes
    }
    if (r < U && !half) node_write<D, SC>(A, m, r, t, sacc);
  }
}
#else
template <int D, int OP, int SC>
__device__ __forceinline__ void tile_phase2(const PipeArgs &A, const unsigned char *m, int U,
                                            int64_t t, int tid, const double *cb,
                                            int nth = kTile) {
  const uint16_t *ptr = reinterpret_cast<const uint16_t *>(m + A.off_ptr);
  const uint16_t *inc = reinterpret_cast<const uint16_t *>(m + A.off_inc);
  const uint16_t *perm = reinterpret_cast<const uint16_t *>(m + A.off_perm);
  const int ntask = FEM_P2_LSPLIT > 0 ? reinterpret_cast<const int *>(m)[3] : 0;
  if (FEM_P2_LSPLIT > 0 && ntask > 0) {  // FEM_P2_LSPLIT tasks: long nodes on lane pairs (warp-uniform loop: shuffles)
    const int nround = (ntask + 31) & ~31;
    for (int q = tid; q < nround; q += nth) {
      const bool act = q < ntask;
      const unsigned tk = act ? perm[q] : 0u;
      const int r = tk & 0xfff;
      const bool first = (tk >> 14) & 1u, second = (tk >> 15) & 1u;
      int lo = 0, hi = 0;
      if (act) {
        lo = ptr[r];
        hi = ptr[r + 1];
        const int mid = (lo + hi + 1) >> 1;
        if (first) hi = mid;
        if (second) lo = mid;
      }
      double s0[D], s1[D];
#pragma unroll
      for (int cc = 0; cc < D; ++cc) s0[cc] = s1[cc] = 0.0;
      int w = lo;
      for (; w + 1 < hi; w += 2) {
        const int p0 = inc[w], p1 = inc[w + 1];
#pragma unroll
        for (int cc = 0; cc < D; ++cc) {
          s0[cc] += cb[p0 + cc * kTile];
          s1[cc] += cb[p1 + cc * kTile];
        }
      }
      if (w < hi) {
        const int pk = inc[w];
#pragma unroll
        for (int cc = 0; cc < D; ++cc) s0[cc] += cb[pk + cc * kTile];
      }
      double sacc[D];
#pragma unroll
      for (int cc = 0; cc < D; ++cc) {
        sacc[cc] = s0[cc] + s1[cc];
        const double oth = __shfl_down_sync(0xffffffffu, sacc[cc], 1);
        if (first) sacc[cc] += oth;   // (first half) + (second half)
      }
      if (act && !second) node_write<D, SC>(A, m, r, t, sacc);
    }
    return;
  }
  for (int q = tid; q < U; q += nth) {  // one thread per tile node, D components
    const int r = A.has_perm ? perm[q] : q;
    const int lo = ptr[r], hi = ptr[r + 1];
    // two interleaved partial sums (even / odd incidences, combined in a fixed order):
    // halves the dependent shared-memory-load -> add chain of the node's sum (A/B at cfg 3:
    // residual 0.86 -> 0.83 ms, HVP 1.056 -> 1.042 ms; 3- and 4-way splits were slower)
    double s0[D], s1[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) s0[cc] = s1[cc] = 0.0;
    int w = lo;
#pragma unroll kP2Unroll
    for (; w + 1 < hi; w += 2) {
      const int p0 = inc[w], p1 = inc[w + 1];
#pragma unroll
      for (int cc = 0; cc < D; ++cc) {
        s0[cc] += cb[p0 + cc * kTile];
        s1[cc] += cb[p1 + cc * kTile];
      }
    }
    if (w < hi) {
      const int pk = inc[w];
#pragma unroll
      for (int cc = 0; cc < D; ++cc) s0[cc] += cb[pk + cc * kTile];
    }
    double sacc[D];
#pragma unroll
    for (int cc = 0; cc < D; ++cc) sacc[cc] = s0[cc] + s1[cc];
    node_write<D, SC>(A, m, r, t, sacc);
  }
}
#endif

// Residual / energy: CTA-wide pipeline (cp.async.wait_all + barrier per tile).  HVP (the
// register-heaviest, 2 CTAs/SM): barrier-free data path — every thread's cp.async copies of
// a stage arrive (cp.async.mbarrier.arrive.noinc) on that stage buffer's mbarrier (expected
// count kTile) and consumers wait on its phase; the only __syncthreads per tile separates
// phase 1 from phase 2, and the contribution array is double-buffered, so threads that
// finish phase 2 of tile k go on to phase 1 of tile k+1 while others are still summing.
// Buffer reuse is ordered by that barrier: tile k+1's node data overwrites tile k-1's (read
// in phase 1 of k-1, before barrier k-1); tile k+2's metadata overwrites tile k-1's (read in
// phase 2 of k-1, before barrier k) and is issued after barrier k.  A/B (profiles/): HVP
// 1.13 -> 1.06 ms; residual / energy slower this way (smem of the second buffer, 3-4 CTAs/SM).
// (mbarrier and TMA bulk-copy helpers: pipe.cuh)

#ifndef FEM_RES_DEC
#define FEM_RES_DEC 0
#endif
// Barrier-free decoupled pipeline: the per-tile __syncthreads between phase 1 and phase 2 is
// replaced by two mbarriers per contribution buffer (phase 1 of tile k done: all threads
// arrive, node-sum threads wait; phase 2 of tile k done: all arrive, the writers of tile
// k+2's contributions / tile k+3's metadata wait), so warps without node sums run up to one
// tile ahead instead of idling at the barrier.  Correct (parity-tested) but measured much
// slower at cfg 3 (HVP 1.69 vs 0.94 ms: the spinning mbarrier waits and the drifted warps'
// buffer waits cost more than the barrier), so off by default.
#ifndef FEM_DEC2
#define FEM_DEC2 0
#endif
// HVP on the mbarrier-decoupled pipeline (double-buffered contributions); 0: the CTA-wide
// pipeline of the residual (single contribution buffer: 60 KB of shared memory at cfg 3, so
// 3 CTAs/SM fit when the register budget allows, FEM_HVP_MINB=3)
#ifndef FEM_HVP_DEC
#define FEM_HVP_DEC 1
#endif
// tile metadata blocks by one TMA bulk copy per tile (thread 0, mbarrier byte count) instead of
// 16-byte cp.async by every thread
#ifndef FEM_TMA_META
#define FEM_TMA_META 1
#endif
#ifndef FEM_ENERGY_DEC
#define FEM_ENERGY_DEC 0
#endif
// metadata buffers of the decoupled (HVP) pipeline: 3 = tile k+2's block issued after barrier
// k; 4 = tile k+3's (ncu r02 source counters: 6.5 % of the HVP's stall samples waiting on the
// next tile's metadata at the top of an iteration — a TMA bulk copy with half an iteration
// of lead time).  Measured (r02, cfg 3, same box, twice): HVP 0.923 / 0.924 ms with 4 buffers
// against 0.910 / 0.911 with 3 (the extra 7 KB per CTA comes out of L1): 3 kept.
#ifndef FEM_META_BUFS
#define FEM_META_BUFS 3
#endif
static_assert(FEM_META_BUFS == 3 || FEM_META_BUFS == 4, "FEM_META_BUFS: 3 or 4");
template <int OP>
constexpr bool pipe_decoupled();
template <int OP>
constexpr int meta_bufs() { return pipe_decoupled<OP>() && !FEM_DEC2 ? FEM_META_BUFS : 3; }
template <int OP>
constexpr bool pipe_decoupled() {
  return (FEM_HVP_DEC && op_is_hvp<OP>() && !op_streams<OP>()) || (FEM_RES_DEC && OP == OP_RESIDUAL) ||
         (FEM_ENERGY_DEC && OP == OP_ENERGY);
}

template <int D, int MAT, int OP, bool MASK, int SC>
__global__ void __launch_bounds__(kTile, pipe_minb(OP, MAT, D)) k_tile_pipe(PipeArgs A) {
  constexpr bool NEED_U = op_needs_u<OP, MAT>();
  constexpr bool NEED_X = op_needs_x<OP, MAT>();
  // node-data slots per stage: x (if read), u (if read), v (HVP)
  constexpr int NF = (NEED_X ? 1 : 0) + (NEED_U ? 1 : 0) + (op_is_hvp<OP>() ? 1 : 0);
  constexpr int UOFF = NEED_X ? 1 : 0;
  constexpr bool DEC = pipe_decoupled<OP>();
  constexpr bool STREAM = op_streams<OP>();
  constexpr unsigned GBYTES = sizeof(double) * geom_words(D) * kTile;
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int NMB = meta_bufs<OP>();
  __shared__ __align__(8) uint64_t mb_meta[4], mb_node[2], mb_geom[2], mb_p1[2], mb_p2[2];
  const int tid = threadIdx.x;
  const int mb = A.mb, um = A.um;
  const int nstride = um * D * NF;
  unsigned char *metab = sm;
  double *nodeb = reinterpret_cast<double *>(sm + NMB * mb);
  double *contrib = nodeb + 2 * nstride;
  constexpr int CBS = cb_stride<OP>();  // contribution row stride (G8: 8 zero pad columns)
  double *geomb = contrib + (DEC ? 2 : 1) * ((D + 1) * D * CBS);  // STREAM: 2 blocks
  const int64_t G = gridDim.x;

  auto tile_id = [&](int64_t i) -> int64_t { return A.list ? (int64_t)__ldg(A.list + i) : i; };
  if constexpr (op_g8<OP>()) {  // the pad columns read by the G8 node sums
    for (int q = tid; q < (DEC ? 2 : 1) * (D + 1) * D * 8; q += kTile)
      contrib[(q / 8) * CBS + kTile + (q % 8)] = 0.0;
  }
  auto issue_geom = [&](int64_t t, int b) {  // one TMA bulk copy of the tile's geometry block
    if (tid == 0) {
      mb_expect_tx(&mb_geom[b], GBYTES);
      bulk_g2s(geomb + b * (GBYTES / 8), A.geom + tile_id(t) * (int64_t)(GBYTES / 8), GBYTES,
               &mb_geom[b]);
    }
  };
  auto issue_meta = [&](int64_t t, int b) {
    unsigned char *dst = metab + b * mb;
    const unsigned char *src = A.meta + tile_id(t) * (int64_t)mb;
    if (FEM_TMA_META) {  // one TMA bulk copy, completion on mb_meta[b] (byte count)
      if (tid == 0) {
        mb_expect_tx(&mb_meta[b], (unsigned)mb);
        bulk_g2s(dst, src, (unsigned)mb, &mb_meta[b]);
      }
    } else {
      for (int off = tid * 16; off < mb; off += kTile * 16) cp_async16(dst + off, src + off);
      if constexpr (DEC) mb_cp_arrive(&mb_meta[b]);
    }
  };
  auto issue_nodes = [&](const unsigned char *m, int b) {
    double *dst = nodeb + b * nstride;
    const int U = reinterpret_cast<const int *>(m)[0];
    const int32_t *nodes = reinterpret_cast<const int32_t *>(m + A.off_nodes);
    if (FEM_ISSUE_NODE) {
      for (int r = tid; r < U; r += kTile) {
        const int64_t g = (int64_t)nodes[r] * D;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          if constexpr (NEED_X) cp_async8(dst + r * D + c, A.coords + g + c);
          if constexpr (NEED_U) cp_async8(dst + UOFF * um * D + r * D + c, A.u + g + c);
          if constexpr (op_is_hvp<OP>()) cp_async8(dst + (NF - 1) * um * D + r * D + c, A.v + g + c);
        }
      }
    } else {
      for (int i = tid; i < U * D; i += kTile) {
        const int64_t g = (int64_t)nodes[i / D] * D + (i % D);
        if constexpr (NEED_X) cp_async8(dst + i, A.coords + g);
        if constexpr (NEED_U) cp_async8(dst + UOFF * um * D + i, A.u + g);
        if constexpr (op_is_hvp<OP>()) cp_async8(dst + (NF - 1) * um * D + i, A.v + g);
      }
    }
    if constexpr (DEC) mb_cp_arrive(&mb_node[b]);
  };

  // OP_*_R: the next tile's reference-metric block (contiguous, refm_words(D) rows) -> L2
  auto prefetch_refm = [&](int64_t tn) {
    if constexpr (op_refm<OP>()) {
      if (tid < refm_words(D)) {
        const double *src = A.refm + (tile_id(tn) * refm_words(D) + tid) * kTile;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src),
                     "r"((unsigned)(kTile * sizeof(double)))
                     : "memory");
      }
    }
  };
  double eacc = 0.0;
  int64_t t = blockIdx.x;
  if (t < A.n_tiles) prefetch_refm(t);
  if constexpr (DEC) {
    if (tid == 0) {
      for (int b = 0; b < NMB; ++b) mb_init(&mb_meta[b], FEM_TMA_META ? 1 : kTile);
      for (int b = 0; b < 2; ++b) mb_init(&mb_node[b], kTile);
      for (int b = 0; b < 2; ++b) mb_init(&mb_p1[b], kTile);
      for (int b = 0; b < 2; ++b) mb_init(&mb_p2[b], kTile);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    for (int b = 0; b < NMB - 1; ++b)
      if (t + b * G < A.n_tiles) issue_meta(t + b * G, b);
    if (t < A.n_tiles) {
      mb_wait(&mb_meta[0], 0);
      issue_nodes(metab, 0);
    }
    if constexpr (FEM_DEC2 && !FEM_P2_BAL) {
      for (int k = 0; t < A.n_tiles; ++k, t += G) {
        const int bm = k % 3, bn = k & 1;
        const unsigned char *m = metab + bm * mb;
        mb_wait(&mb_node[bn], (unsigned)(k >> 1) & 1u);  // node data of tile k
        if (t + G < A.n_tiles) {  // node data of tile k+1 -> buffer of tile k-1
          const int bm1 = (k + 1) % 3;
          mb_wait(&mb_meta[bm1], (unsigned)((k + 1) / 3) & 1u);
          if (k >= 1) mb_wait(&mb_p1[(k - 1) & 1], (unsigned)((k - 1) >> 1) & 1u);
          issue_nodes(metab + bm1 * mb, bn ^ 1);
          if constexpr (OP == OP_HVP_LIN && MAT == FEM_NEO_HOOKEAN) {  // cache rows of tile k+1 -> L2
            if (tid < lin_words(D)) {
              const double *src = A.lin + tid * A.lin_stride + tile_id(t + G) * kTile;
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src),
                           "r"((unsigned)(kTile * sizeof(double)))
                           : "memory");
            }
          }
          prefetch_refm(t + G);
        }
        const double *nb = nodeb + bn * nstride;
        double *cb = contrib + (k & 1) * ((D + 1) * D * CBS);
        if (k >= 2) mb_wait(&mb_p2[k & 1], (unsigned)((k - 2) >> 1) & 1u);  // tile k-2 summed
        tile_phase1<D, MAT, OP, MASK>(A, m, nb, nb + UOFF * um * D, nb + (NF - 1) * um * D, tile_id(t), tid, cb, eacc);
        mb_arrive(&mb_p1[k & 1]);
        if (t + 2 * G < A.n_tiles) {  // metadata of tile k+2 -> buffer of tile k-1
          if (k >= 1) mb_wait(&mb_p2[(k - 1) & 1], (unsigned)((k - 1) >> 1) & 1u);
          issue_meta(t + 2 * G, (k + 2) % 3);
        }
        const int U = reinterpret_cast<const int *>(m)[0];
        const int nt2 = FEM_P2_LSPLIT > 0 ? reinterpret_cast<const int *>(m)[3] : 0;  // FEM_P2_LSPLIT tasks
        if (tid < (FEM_P2_PAIR ? 2 * U : nt2 > 0 ? ((nt2 + 31) & ~31) : U))
          mb_wait(&mb_p1[k & 1], (unsigned)(k >> 1) & 1u);  // all of tile k's phase 1
        if constexpr (op_g8<OP>()) tile_phase2_g8<D, OP, SC>(A, m, U, tile_id(t), tid, cb);
        else if constexpr (op_has_p2<OP>()) tile_phase2<D, OP, SC>(A, m, U, tile_id(t), tid, cb);
        mb_arrive(&mb_p2[k & 1]);
      }
    } else {
      for (int k = 0; t < A.n_tiles; ++k, t += G) {
        const int bm = k % NMB, bn = k & 1;
        const unsigned char *m = metab + bm * mb;
        mb_wait(&mb_node[bn], (unsigned)(k >> 1) & 1u);  // node data of tile k
        if (t + G < A.n_tiles) {  // node data of tile k+1 (its metadata issued after barrier k+2-NMB)
          const int bm1 = (k + 1) % NMB;
          mb_wait(&mb_meta[bm1], (unsigned)((k + 1) / NMB) & 1u);
          issue_nodes(metab + bm1 * mb, bn ^ 1);
          if constexpr (OP == OP_HVP_LIN && MAT == FEM_NEO_HOOKEAN) {  // cache rows of tile k+1 -> L2
            if (tid < lin_words(D)) {
              const double *src = A.lin + tid * A.lin_stride + tile_id(t + G) * kTile;
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src),
                           "r"((unsigned)(kTile * sizeof(double)))
                           : "memory");
            }
          }
          prefetch_refm(t + G);
        }
        const double *nb = nodeb + bn * nstride;
        double *cb = contrib + (k & 1) * ((D + 1) * D * CBS);
        tile_phase1<D, MAT, OP, MASK>(A, m, nb, nb + UOFF * um * D, nb + (NF - 1) * um * D, tile_id(t), tid, cb, eacc);
        __syncthreads();  // phase 1 of tile k done; tile k-1 fully consumed
        if (t + (NMB - 1) * G < A.n_tiles) issue_meta(t + (NMB - 1) * G, (k + NMB - 1) % NMB);
        if constexpr (op_g8<OP>())
          tile_phase2_g8<D, OP, SC>(A, m, reinterpret_cast<const int *>(m)[0], tile_id(t), tid, cb);
        else if constexpr (op_has_p2<OP>())
          tile_phase2<D, OP, SC>(A, m, reinterpret_cast<const int *>(m)[0], tile_id(t), tid, cb);
      }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  } else {
    if (STREAM || FEM_TMA_META) {
      if (tid == 0) {
        for (int b = 0; b < 2; ++b) mb_init(&mb_geom[b], 1);
        for (int b = 0; b < 3; ++b) mb_init(&mb_meta[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      }
      __syncthreads();
    }
    if (t < A.n_tiles) {
      issue_meta(t, 0);
      cp_async_commit();
      cp_async_wait_all();
      if (FEM_TMA_META) mb_wait(&mb_meta[0], 0);
      __syncthreads();
      issue_nodes(metab, 0);
      if constexpr (STREAM) issue_geom(t, 0);
      if (t + G < A.n_tiles) issue_meta(t + G, 1);
      cp_async_commit();
    }
    for (int k = 0; t < A.n_tiles; ++k, t += G) {
      cp_async_wait_all();
      __syncthreads();
      if constexpr (STREAM) mb_wait(&mb_geom[k & 1], (unsigned)(k >> 1) & 1u);
      const unsigned char *m = metab + (k % 3) * mb;
      const double *nb = nodeb + (k & 1) * nstride;
      if (t + G < A.n_tiles) {
        if (FEM_TMA_META) mb_wait(&mb_meta[(k + 1) % 3], (unsigned)((k + 1) / 3) & 1u);
        issue_nodes(metab + ((k + 1) % 3) * mb, (k + 1) & 1);
        if constexpr (STREAM) issue_geom(t + G, (k + 1) & 1);
        prefetch_refm(t + G);
      }
      if (t + 2 * G < A.n_tiles) issue_meta(t + 2 * G, (k + 2) % 3);
      cp_async_commit();
      tile_phase1<D, MAT, OP, MASK>(A, m, nb, nb + UOFF * um * D, nb + (NF - 1) * um * D, tile_id(t), tid, contrib, eacc,
                                    STREAM ? geomb + (k & 1) * (GBYTES / 8) : nullptr);
      if constexpr (op_has_p2<OP>()) {
        __syncthreads();
        if constexpr (op_g8<OP>())
          tile_phase2_g8<D, OP, SC>(A, m, reinterpret_cast<const int *>(m)[0], tile_id(t), tid, contrib);
        else
          tile_phase2<D, OP, SC>(A, m, reinterpret_cast<const int *>(m)[0], tile_id(t), tid, contrib);
      }
      __syncthreads();
    }
  }
  if (OP == OP_ENERGY || (OP == OP_RESIDUAL && A.partials)) {  // uniform over the CTA
    const double tsum = block_sum<kTile>(eacc);
    if (tid == 0) A.partials[blockIdx.x] = tsum;
  }
}


// ------------------------------------------------------------------ warp-specialized tiles
// FEM_WS: residual / HVP with the roles split by warpgroup (setmaxnreg): warpgroups 0-1 (one
// element per thread) run only phase 1; warpgroup 2 (the producer) stages every tile — its
// metadata block by one TMA bulk copy, its nodal data by cp.async gathers — and runs phase 2
// (the node sums and writes) of tile k while the element warps compute tile k+1.  Hand-offs
// are mbarriers: node[b] (data landed, 128 producer arrivals), full[b] (phase 1 done, 256),
// empty[b] (contributions consumed, 128); contributions and node data double-buffered, the
// metadata triple-buffered.  No CTA-wide barrier in the loop, so the element warps never
// wait for the node sums (the ~24 % barrier stall of k_tile_pipe).  Registers: launch 80 x
// 384; the producer gives back to 48, the element warps take 96.  Parity-tested; measured at
// cfg 3 (r02, same box): HVP 0.984 / residual 0.845 ms against 0.925 / 0.795 for k_tile_pipe
// (producer 32 / elements 104 registers: 1.155 / 1.037 — the node sums serialise their loads;
// three contribution buffers: 1.123 / 0.930).  ncu: the element warps now wait on empty[b]
// (25 % of stall samples): the producer's latency-bound node sums, stretched by issue
// contention with 16 element warps, take longer than phase 1 — so off by default.
#ifndef FEM_WS_RC
#define FEM_WS_RC 96
#endif
#ifndef FEM_WS_RP
#define FEM_WS_RP 48
#endif
#ifndef FEM_WS_CB
#define FEM_WS_CB 2   // contribution buffers (the element warps run up to CB tiles ahead)
#endif
constexpr int kWsProd = 128;  // producer threads (one warpgroup)
static_assert(kTile == 256, "FEM_WS: two element warpgroups per 256-element tile");

template <int D, int MAT, int OP, bool MASK>
__global__ void __launch_bounds__(kTile + kWsProd, 2) k_tile_ws(PipeArgs A) {
  constexpr bool NEED_U = op_needs_u<OP, MAT>();
  constexpr bool NEED_X = op_needs_x<OP, MAT>();
  constexpr int NF = (NEED_X ? 1 : 0) + (NEED_U ? 1 : 0) + (op_is_hvp<OP>() ? 1 : 0);
  constexpr int UOFF = NEED_X ? 1 : 0;
  constexpr int CB = (D + 1) * D * kCbStride;
  constexpr int NCB = FEM_WS_CB;
  static_assert(!FEM_WS || (!FEM_P2_BAL && !FEM_P2_NM && !FEM_P2_G8 && !FEM_P2_PAIR), "FEM_WS: default phase 2");
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t mb_meta[3], mb_node[2], mb_full[NCB], mb_empty[NCB];
  const int tid = threadIdx.x;
  const int mb = A.mb, um = A.um;
  const int nstride = um * D * NF;
  unsigned char *metab = sm;
  double *nodeb = reinterpret_cast<double *>(sm + 3 * mb);
  double *contrib = nodeb + 2 * nstride;
  const int64_t G = gridDim.x, t0 = blockIdx.x;
  const int64_t nk = t0 < A.n_tiles ? (A.n_tiles - 1 - t0) / G + 1 : 0;  // tiles of this CTA
  auto tile_id = [&](int64_t k) -> int64_t {
    const int64_t i = t0 + k * G;
    return A.list ? (int64_t)__ldg(A.list + i) : i;
  };
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mb_init(&mb_meta[b], 1);
    for (int b = 0; b < 2; ++b) mb_init(&mb_node[b], kWsProd);
    for (int b = 0; b < NCB; ++b) {
      mb_init(&mb_full[b], kTile);
      mb_init(&mb_empty[b], kWsProd);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid >= kTile) {  // ---------------- producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(FEM_WS_RP) : "memory");
    const int pt = tid - kTile;
    auto issue_meta = [&](int64_t k) {
      if (pt == 0) {
        uint64_t *bar = &mb_meta[k % 3];
        mb_expect_tx(bar, (unsigned)mb);
        bulk_g2s(metab + (k % 3) * mb, A.meta + tile_id(k) * (int64_t)mb, (unsigned)mb, bar);
      }
    };
    auto issue_nodes = [&](int64_t k) {  // tile k's nodal data -> node buffer k & 1
      const unsigned char *m = metab + (k % 3) * mb;
      double *dst = nodeb + (k & 1) * nstride;
      const int U = reinterpret_cast<const int *>(m)[0];
      const int32_t *nodes = reinterpret_cast<const int32_t *>(m + A.off_nodes);
      for (int r = pt; r < U; r += kWsProd) {
        const int64_t g = (int64_t)nodes[r] * D;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          if constexpr (NEED_X) cp_async8(dst + r * D + c, A.coords + g + c);
          if constexpr (NEED_U) cp_async8(dst + UOFF * um * D + r * D + c, A.u + g + c);
          if constexpr (op_is_hvp<OP>()) cp_async8(dst + (NF - 1) * um * D + r * D + c, A.v + g + c);
        }
      }
      mb_cp_arrive(&mb_node[k & 1]);
    };
    for (int64_t k = 0; k < 3 && k < nk; ++k) issue_meta(k);
    for (int64_t k = 0; k < 2 && k < nk; ++k) {
      mb_wait(&mb_meta[k % 3], (unsigned)(k / 3) & 1u);
      issue_nodes(k);
    }
    for (int64_t k = 0; k < nk; ++k) {
      mb_wait(&mb_full[k % NCB], (unsigned)(k / NCB) & 1u);  // phase 1 of tile k done
      if (k + 2 < nk) {  // node buffer k & 1 is free: tile k + 2's data
        mb_wait(&mb_meta[(k + 2) % 3], (unsigned)((k + 2) / 3) & 1u);
        issue_nodes(k + 2);
      }
      const unsigned char *m = metab + (k % 3) * mb;
      tile_phase2<D, OP, 0>(A, m, reinterpret_cast<const int *>(m)[0], tile_id(k), pt,
                            contrib + (k % NCB) * CB, kWsProd);
      mb_arrive(&mb_empty[k % NCB]);
      asm volatile("bar.sync 1, %0;\n" ::"n"(kWsProd) : "memory");  // metadata k read by all
      if (k + 3 < nk) issue_meta(k + 3);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  } else {  // ---------------- element warpgroups
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(FEM_WS_RC) : "memory");
    double eacc = 0.0;
    for (int64_t k = 0; k < nk; ++k) {
      mb_wait(&mb_node[k & 1], (unsigned)(k >> 1) & 1u);                     // tile k staged
      if (k >= NCB) mb_wait(&mb_empty[k % NCB], (unsigned)((k - NCB) / NCB) & 1u);  // buffer free
      const unsigned char *m = metab + (k % 3) * mb;
      const double *nb = nodeb + (k & 1) * nstride;
      tile_phase1<D, MAT, OP, MASK>(A, m, nb, nb + UOFF * um * D, nb + (NF - 1) * um * D,
                                    tile_id(k), tid, contrib + (k % NCB) * CB, eacc);
      mb_arrive(&mb_full[k % NCB]);
    }
  }
}

// DET: y[node] = sum of its tile slots in tile order
template <int D>
__global__ void k_slot_gather(const int64_t *node_slot_ptr, const int32_t *node_slots,
                              const double *slots, int64_t n_nodes, double *out) {
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    double s[D];
#pragma unroll
    for (int c = 0; c < D; ++c) s[c] = 0.0;
    for (int64_t q = node_slot_ptr[n]; q < node_slot_ptr[n + 1]; ++q) {
      const int64_t sl = node_slots[q];
#pragma unroll
      for (int c = 0; c < D; ++c) s[c] += slots[sl * D + c];
    }
#pragma unroll
    for (int c = 0; c < D; ++c) out[n * D + c] = s[c];
  }
}

// grid of the persistent kernels (fixed per problem: deterministic energy partial order)
// grid of the persistent kernels: 148 SMs x CTAs/SM of the op (fixed per problem and op,
// so the energy partial order is deterministic)
static int pipe_grid(Problem *p, int op, int64_t n = -1) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(n < 0 ? p->tiles.n_tiles : n, 148 * pipe_minb(op, p->material, p->dim)));
}

template <int D, int MAT, int OP, bool MASK, int SC>
static fem_status launch_pipe_t(Problem *p, const PipeArgs &a, cudaStream_t s) {
  const TileSet &T = p->tiles;
  const bool need_u = op_needs_u<OP, MAT>();
  const int nf = (op_needs_x<OP, MAT>() ? 1 : 0) + (need_u ? 1 : 0) + (op_is_hvp<OP>() ? 1 : 0);
  if constexpr (op_refm<OP>()) static_assert(MAT == FEM_NEO_HOOKEAN, "OP_*_R: neo-Hookean only");
  const size_t smem = (size_t)meta_bufs<OP>() * (op_g8<OP>() ? T.mb_g8 : T.mb) + sizeof(double) * 2 * (size_t)T.um * D * nf +
                      (!op_has_p2<OP>() ? 0 : (pipe_decoupled<OP>() ? 2 : 1) * sizeof(double) * (size_t)(D + 1) * D * cb_stride<OP>()) +
                      (op_streams<OP>() ? 2 * sizeof(double) * geom_words(D) * kTile : 0);
  auto kern = k_tile_pipe<D, MAT, OP, MASK, SC>;
  FEM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<pipe_grid(p, OP, a.n_tiles), kTile, smem, s>>>(a);
  FEM_LAUNCH_CHECK("tile pipeline kernel");
  return FEM_OK;
}

template <int D, int MAT, int OP, bool MASK>
static fem_status launch_ws_t(Problem *p, const PipeArgs &a, cudaStream_t s) {
  const TileSet &T = p->tiles;
  const int nf = (op_needs_x<OP, MAT>() ? 1 : 0) + (op_needs_u<OP, MAT>() ? 1 : 0) + (op_is_hvp<OP>() ? 1 : 0);
  const size_t smem = (size_t)3 * T.mb + sizeof(double) * 2 * (size_t)T.um * D * nf +
                      FEM_WS_CB * sizeof(double) * (size_t)(D + 1) * D * kCbStride;
  auto kern = k_tile_ws<D, MAT, OP, MASK>;
  FEM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.n_tiles, 148 * 2));
  kern<<<grid, kTile + kWsProd, smem, s>>>(a);
  FEM_LAUNCH_CHECK("warp-specialized tile kernel");
  return FEM_OK;
}

template <int OP, bool MASK>
static fem_status launch_ws_op(Problem *p, const PipeArgs &a, cudaStream_t s) {
  if (p->dim == 2) {
    if (p->material == FEM_LINEAR_ELASTIC) return launch_ws_t<2, FEM_LINEAR_ELASTIC, OP, MASK>(p, a, s);
    return launch_ws_t<2, FEM_NEO_HOOKEAN, OP, MASK>(p, a, s);
  }
  if (p->material == FEM_LINEAR_ELASTIC) return launch_ws_t<3, FEM_LINEAR_ELASTIC, OP, MASK>(p, a, s);
  return launch_ws_t<3, FEM_NEO_HOOKEAN, OP, MASK>(p, a, s);
}

template <int OP, bool MASK, int SC>
static fem_status launch_pipe_op(Problem *p, const PipeArgs &a, cudaStream_t s) {
  if constexpr (op_refm<OP>()) {  // neo-Hookean only (tile_pass maps LE to the base op)
    if (p->dim == 2) return launch_pipe_t<2, FEM_NEO_HOOKEAN, OP, MASK, SC>(p, a, s);
    return launch_pipe_t<3, FEM_NEO_HOOKEAN, OP, MASK, SC>(p, a, s);
  } else {
    if (p->dim == 2) {
      if (p->material == FEM_LINEAR_ELASTIC) return launch_pipe_t<2, FEM_LINEAR_ELASTIC, OP, MASK, SC>(p, a, s);
      return launch_pipe_t<2, FEM_NEO_HOOKEAN, OP, MASK, SC>(p, a, s);
    }
    if (p->material == FEM_LINEAR_ELASTIC) return launch_pipe_t<3, FEM_LINEAR_ELASTIC, OP, MASK, SC>(p, a, s);
    return launch_pipe_t<3, FEM_NEO_HOOKEAN, OP, MASK, SC>(p, a, s);
  }
}

// Streamed geometry (FEM_STREAM_GEOM): per tile one contiguous SoA block {c_a[j] (D x D),
// det J} x kTile elements in tile order, computed once from the coordinates (same cofactor
// arithmetic as the recompute path), loaded per tile by one TMA bulk copy.
template <int D>
__global__ void k_geom_stream(const double *coords, const int32_t *conn, const int32_t *perm,
                              int64_t E, int64_t n_slots, double *geom) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_slots;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / kTile, l = i % kTile;
    double *g = geom + t * geom_words(D) * kTile + l;
    if (i >= E) {
      for (int w = 0; w < D * D; ++w) g[w * kTile] = 0.0;
      g[D * D * kTile] = 1.0;
      continue;
    }
    const int64_t e = perm[i];
    double x[D + 1][D], c[D][D];
    for (int a = 0; a <= D; ++a)
      for (int j = 0; j < D; ++j) x[a][j] = coords[(int64_t)conn[e * (D + 1) + a] * D + j];
    const double det = cof_gradients<D>(x, c);
    for (int a = 0; a < D; ++a)
      for (int j = 0; j < D; ++j) g[(a * D + j) * kTile] = c[a][j];
    g[D * D * kTile] = det;
  }
}

// Reference metric (OP_*_R): per tile one contiguous SoA block {mu vol G_a.G_b (a <= b),
// 1/det J} x kTile elements in tile order, computed once per problem from the coordinates with
// the recompute path's own arithmetic (cofactors, fem_rcp, sr = mu id / d!), so the cached and
// recomputed kernels see the same bits.  mu is the element's (phase table) shear modulus.
template <int D>
__global__ void k_refm(const double *coords, const int32_t *conn, const int32_t *perm,
                       const uint8_t *phase, const double *mu_tab, double mu0, int64_t E,
                       int64_t n_slots, double *refm) {
  constexpr int RW = refm_words(D);
  constexpr double inv_fact = (D == 3) ? 1.0 / 6.0 : 0.5;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_slots;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / kTile, l = i % kTile;
    double *g = refm + t * RW * kTile + l;
    if (i >= E) {
      for (int w = 0; w < RW - 1; ++w) g[w * kTile] = 0.0;
      g[(RW - 1) * kTile] = 1.0;
      continue;
    }
    const int64_t e = perm[i];
    double x[D + 1][D], c[D][D];
    for (int a = 0; a <= D; ++a)
      for (int j = 0; j < D; ++j) x[a][j] = coords[(int64_t)conn[e * (D + 1) + a] * D + j];
    const double det = cof_gradients<D>(x, c);
    const double id = fem_rcp(det);
    const double mu = phase ? mu_tab[phase[i]] : mu0;
    const double sr = mu * id * inv_fact;
    for (int a = 0; a < D; ++a)
      for (int b = a; b < D; ++b) {
        double tt = 0.0;
        for (int j = 0; j < D; ++j) tt = fma(c[a][j], c[b][j], tt);
        g[sym_idx(a, b, D) * kTile] = sr * tt;
      }
    g[(RW - 1) * kTile] = id;
  }
}

fem_status build_refm(Problem *p, cudaStream_t s) {
  TileSet &T = p->tiles;
  if (T.refm) return FEM_OK;
  const int D = p->dim;
  const int64_t n_slots = T.n_tiles * kTile;
  FEM_CUDA(cudaMalloc(&T.refm, sizeof(double) * refm_words(D) * n_slots));
  if (D == 3) k_refm<3><<<grid_for(n_slots), kThreads, 0, s>>>(p->coords, p->conn, T.perm, T.phase, p->mu_tab, p->mu, p->n_elems, n_slots, T.refm);
  else k_refm<2><<<grid_for(n_slots), kThreads, 0, s>>>(p->coords, p->conn, T.perm, T.phase, p->mu_tab, p->mu, p->n_elems, n_slots, T.refm);
  FEM_LAUNCH_CHECK("reference metric");
  return FEM_OK;
}

fem_status build_geom_stream(Problem *p, cudaStream_t s) {
  TileSet &T = p->tiles;
  if (T.geom) return FEM_OK;
  const int D = p->dim;
  const int64_t n_slots = T.n_tiles * kTile;
  FEM_CUDA(cudaMalloc(&T.geom, sizeof(double) * geom_words(D) * n_slots));
  if (D == 3) k_geom_stream<3><<<grid_for(n_slots), kThreads, 0, s>>>(p->coords, p->conn, T.perm, p->n_elems, n_slots, T.geom);
  else k_geom_stream<2><<<grid_for(n_slots), kThreads, 0, s>>>(p->coords, p->conn, T.perm, p->n_elems, n_slots, T.geom);
  FEM_LAUNCH_CHECK("geometry stream");
  return FEM_OK;
}

// Tile coloring (FEM_TILE_COLORED): greedy in tile (Morton) order, a tile takes the smallest
// color none of its nodes' earlier tiles holds (per-node 128-bit masks over the tiles' node
// lists, a host pass at setup).  Tiles of one color share no node, so a pass over them
// writes the tile-boundary sums with plain read-add-write: the color-ordered conflict-free
// scatter at tile granularity (each tile keeps its in-tile reduction and its locality).
fem_status build_tile_colors(Problem *p, cudaStream_t s) {
  TileSet &T = p->tiles;
  if (T.tcolor_list) return FEM_OK;
  const int64_t nt = T.n_tiles;
  std::vector<int32_t> U(nt), nodes((size_t)nt * T.maxe);
  FEM_CUDA(cudaMemcpyAsync(U.data(), T.U, sizeof(int32_t) * nt, cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaMemcpyAsync(nodes.data(), T.nodes, sizeof(int32_t) * nodes.size(), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  std::vector<uint64_t> mask((size_t)p->n_nodes * 2, 0ull);
  std::vector<uint8_t> col(nt);
  std::vector<int64_t> cnt(129, 0);
  int nc = 0;
  for (int64_t t = 0; t < nt; ++t) {
    uint64_t m0 = 0, m1 = 0;
    const int32_t *nd = nodes.data() + t * T.maxe;
    for (int r = 0; r < U[t]; ++r) {
      m0 |= mask[2 * (int64_t)nd[r]];
      m1 |= mask[2 * (int64_t)nd[r] + 1];
    }
    const int c = ~m0 ? __builtin_ctzll(~m0) : (~m1 ? 64 + __builtin_ctzll(~m1) : 128);
    if (c >= 128) {
      set_error("FEM_TILE_COLORED: more than 128 tile colors");
      return FEM_ERR_TOO_MANY_COLORS;
    }
    for (int r = 0; r < U[t]; ++r) mask[2 * (int64_t)nd[r] + (c >> 6)] |= 1ull << (c & 63);
    col[t] = (uint8_t)c;
    ++cnt[c + 1];
    nc = std::max(nc, c + 1);
  }
  T.tcolor_off.assign(nc + 1, 0);
  for (int c = 0; c < nc; ++c) T.tcolor_off[c + 1] = T.tcolor_off[c] + cnt[c + 1];
  std::vector<int32_t> list(nt);
  std::vector<int64_t> fill(T.tcolor_off.begin(), T.tcolor_off.end() - 1);
  for (int64_t t = 0; t < nt; ++t) list[fill[col[t]]++] = (int32_t)t;
  FEM_CUDA(cudaMalloc(&T.tcolor_list, sizeof(int32_t) * (nt > 0 ? nt : 1)));
  FEM_CUDA(cudaMemcpyAsync(T.tcolor_list, list.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  return FEM_OK;
}

// Element pass of the residual / HVP (op = OP_RESIDUAL / OP_HVP) or the energy partials
// (OP_ENERGY: one partial per CTA into `partials`, *n_partials set).
fem_status tile_pass(Problem *p, int op, const double *u, const double *v, double *out,
                     bool mask, bool det, double *partials, cudaStream_t s, int part) {
  fem_status st = build_tiles(p, s);
  if (st) return st;
  if (p->n_elems == 0) return FEM_OK;
  if (op == OP_RESIDUAL_R || op == OP_HVP_R) {
    // the reference-metric forms exist for the neo-Hookean spatial kernels; the deterministic
    // slot mode, the tile-colored passes and the energy partials keep the recompute form
    if (p->material != FEM_NEO_HOOKEAN || det || part == 3 || partials)
      op = op == OP_RESIDUAL_R ? OP_RESIDUAL : OP_HVP;
    else {
      st = build_refm(p, s);
      if (st) return st;
    }
  }
  const TileSet &T = p->tiles;
  PipeArgs a{};
  a.meta = T.meta;
  a.n_tiles = T.n_tiles;
  if (part == 1 || part == 2) {  // one of the two halves of TileSet::list (no DET, no energy)
    if (T.n_boundary < 0 || det || op == OP_ENERGY) return FEM_ERR_INVALID_ARG;
    a.list = T.list + (part == 1 ? 0 : T.n_boundary);
    a.n_tiles = part == 1 ? T.n_boundary : T.n_tiles - T.n_boundary;
    if (a.n_tiles == 0) return FEM_OK;
  }
  a.E = p->n_elems;
  a.mb = T.mb; a.um = T.um; a.off_nodes = T.off_nodes; a.off_lconn = T.off_lconn;
  a.off_ptr = T.off_ptr; a.off_inc = T.off_inc; a.off_int = T.off_int; a.off_bc = T.off_bc;
  a.off_ph = T.off_ph;
  a.off_soff = T.off_soff;
  a.off_smeta = T.off_smeta;
  a.off_perm = T.off_perm;
  a.has_phase = T.phase != nullptr;
  a.has_perm = T.p2perm != nullptr;
  // the HVP kernels read the G8 metadata layout (op_g8): same tiles, nodes and lconn offsets
  if (!FEM_P2_G8 && op_g8<OP_HVP>() && op == OP_HVP) {
    if (!T.meta_g8) {
      set_error("HVP tile metadata (G8 layout) missing");
      return FEM_ERR_CUDA;
    }
    a.meta = T.meta_g8;
    a.mb = T.mb_g8;
    a.off_inc = T.off_inc_g8;
    a.off_int = T.off_int_g8;
    a.off_bc = T.off_bc_g8;
    a.off_ph = T.off_ph_g8;
    a.off_perm = T.off_perm_g8;
    a.has_perm = false;
  }
  a.slot_off = T.slot_off;
  a.coords = p->coords;
  a.u = u;
  a.v = v;
  a.lam = p->lam;
  a.mu = p->mu;
  a.lam_tab = p->lam_tab;
  a.mu_tab = p->mu_tab;
  a.out = out;
  a.partials = partials;
  a.err = p->d_err;
  a.lin = p->lin;
  a.lin_stride = T.n_tiles * kTile;
  a.geom = T.geom;
  a.refm = T.refm;
  if (part == 3) {  // tile-colored passes (FEM_TILE_COLORED): plain writes, no atomics
    if (det || (op != OP_RESIDUAL && op != OP_HVP)) return FEM_ERR_INVALID_ARG;
    st = build_tile_colors(p, s);
    if (st) return st;
    for (size_t c = 0; c + 1 < T.tcolor_off.size(); ++c) {
      a.list = T.tcolor_list + T.tcolor_off[c];
      a.n_tiles = T.tcolor_off[c + 1] - T.tcolor_off[c];
      if (op == OP_RESIDUAL) st = launch_pipe_op<OP_RESIDUAL, false, 2>(p, a, s);
      else st = mask ? launch_pipe_op<OP_HVP, true, 2>(p, a, s) : launch_pipe_op<OP_HVP, false, 2>(p, a, s);
      if (st) return st;
    }
    return FEM_OK;
  }
  if (op == OP_ENERGY) return launch_pipe_op<OP_ENERGY, false, 0>(p, a, s);
  if (op == OP_LIN) return launch_pipe_op<OP_LIN, false, 0>(p, a, s);
  if (det) {
    st = ensure(p->slotbuf, sizeof(double) * T.n_slots * p->dim);
    if (st) return st;
    a.slots = (double *)p->slotbuf.ptr;
    if (op == OP_RESIDUAL) st = launch_pipe_op<OP_RESIDUAL, false, 1>(p, a, s);
    else if (op == OP_HVP_LIN) st = mask ? launch_pipe_op<OP_HVP_LIN, true, 1>(p, a, s) : launch_pipe_op<OP_HVP_LIN, false, 1>(p, a, s);
    else st = mask ? launch_pipe_op<OP_HVP, true, 1>(p, a, s) : launch_pipe_op<OP_HVP, false, 1>(p, a, s);
    if (st) return st;
    if (p->dim == 2)
      k_slot_gather<2><<<grid_for(p->n_nodes), kThreads, 0, s>>>(T.node_slot_ptr, T.node_slots, a.slots, p->n_nodes, out);
    else
      k_slot_gather<3><<<grid_for(p->n_nodes), kThreads, 0, s>>>(T.node_slot_ptr, T.node_slots, a.slots, p->n_nodes, out);
    FEM_LAUNCH_CHECK("slot gather");
    return FEM_OK;
  }
  if (op == OP_RESIDUAL_S || op == OP_HVP_S) {
    st = build_geom_stream(p, s);
    if (st) return st;
    a.geom = T.geom;
    if (op == OP_RESIDUAL_S) return launch_pipe_op<OP_RESIDUAL_S, false, 0>(p, a, s);
    return mask ? launch_pipe_op<OP_HVP_S, true, 0>(p, a, s) : launch_pipe_op<OP_HVP_S, false, 0>(p, a, s);
  }
  if (op == OP_RESIDUAL_R) return launch_pipe_op<OP_RESIDUAL_R, false, 0>(p, a, s);
  if (op == OP_HVP_R)
    return mask ? launch_pipe_op<OP_HVP_R, true, 0>(p, a, s) : launch_pipe_op<OP_HVP_R, false, 0>(p, a, s);
  if (FEM_WS && (op == OP_RESIDUAL || op == OP_HVP) && !partials) {
    if (op == OP_RESIDUAL) return launch_ws_op<OP_RESIDUAL, false>(p, a, s);
    return mask ? launch_ws_op<OP_HVP, true>(p, a, s) : launch_ws_op<OP_HVP, false>(p, a, s);
  }
  if (op == OP_RESIDUAL) return launch_pipe_op<OP_RESIDUAL, false, 0>(p, a, s);
  if (op == OP_HVP_LIN)
    return mask ? launch_pipe_op<OP_HVP_LIN, true, 0>(p, a, s) : launch_pipe_op<OP_HVP_LIN, false, 0>(p, a, s);
  return mask ? launch_pipe_op<OP_HVP, true, 0>(p, a, s) : launch_pipe_op<OP_HVP, false, 0>(p, a, s);
}

int tile_energy_partials(Problem *p, int op) { return pipe_grid(p, op); }

__global__ void k_tile_shared(TileSet T, const uint8_t *shared, uint8_t *flag) {
  for (int64_t t = blockIdx.x; t < T.n_tiles; t += gridDim.x) {
    const int U = T.U[t];
    int any = 0;
    for (int r = threadIdx.x; r < U; r += blockDim.x) any |= shared[T.nodes[t * T.maxe + r]];
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) flag[t] = (uint8_t)(any != 0);
  }
}

// Multi-GPU: order the tiles as (tiles touching interface nodes, the rest); stable in tile
// order within each part.
fem_status build_tile_lists(Problem *p, cudaStream_t s) {
  TileSet &T = p->tiles;
  if (T.n_boundary >= 0 || p->size <= 1 || !p->shared) return FEM_OK;
  fem_status st = build_tiles(p, s);
  if (st) return st;
  uint8_t *flag = nullptr;
  FEM_CUDA(cudaMalloc(&flag, T.n_tiles > 0 ? T.n_tiles : 1));
  if (T.n_tiles) k_tile_shared<<<grid_for(T.n_tiles, 1, 148 * 16), 128, 0, s>>>(T, p->shared, flag);
  FEM_LAUNCH_CHECK("tile lists");
  std::vector<uint8_t> hf(T.n_tiles);
  FEM_CUDA(cudaMemcpyAsync(hf.data(), flag, T.n_tiles, cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  cudaFree(flag);
  std::vector<int32_t> lst;
  lst.reserve(T.n_tiles);
  for (int64_t t = 0; t < T.n_tiles; ++t) if (hf[t]) lst.push_back((int32_t)t);
  const int64_t nb = (int64_t)lst.size();
  for (int64_t t = 0; t < T.n_tiles; ++t) if (!hf[t]) lst.push_back((int32_t)t);
  FEM_CUDA(cudaMalloc(&T.list, sizeof(int32_t) * (lst.empty() ? 1 : lst.size())));
  if (!lst.empty()) FEM_CUDA(cudaMemcpyAsync(T.list, lst.data(), sizeof(int32_t) * lst.size(), cudaMemcpyHostToDevice, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  T.n_boundary = nb;
  return FEM_OK;
}


template <int D>
__global__ void k_node_morton(const double *coords, int64_t n, double3 lo, double3 scale,
                              uint64_t *keys, int32_t *idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double l[3] = {lo.x, lo.y, lo.z}, sc[3] = {scale.x, scale.y, scale.z};
    uint64_t q[3] = {0, 0, 0};
    for (int c = 0; c < D; ++c) q[c] = (uint64_t)fmax(0.0, (coords[i * D + c] - l[c]) * sc[c]);
    keys[i] = (D == 3) ? (spread3(q[0]) | spread3(q[1]) << 1 | spread3(q[2]) << 2)
                       : (spread2(q[0]) | spread2(q[1]) << 1);
    idx[i] = (int32_t)i;
  }
}

// Morton order of the nodes (assembly row order), stable sort of centroid-free keys.
fem_status morton_node_order(Problem *p, cudaStream_t s) {
  if (p->node_order || p->n_nodes == 0) return FEM_OK;
  const int D = p->dim;
  const int nb = grid_for(p->n_nodes, kThreads, 256);
  double *part = nullptr;
  FEM_CUDA(cudaMalloc(&part, sizeof(double) * nb * 6));
  k_bbox_partial<<<nb, kThreads, 0, s>>>(p->coords, p->n_nodes, D, part);
  std::vector<double> hp(nb * 6);
  FEM_CUDA(cudaMemcpyAsync(hp.data(), part, sizeof(double) * nb * 6, cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  cudaFree(part);
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int b = 0; b < nb; ++b)
    for (int c = 0; c < 3; ++c) {
      lo[c] = std::min(lo[c], hp[b * 6 + c]);
      hi[c] = std::max(hi[c], hp[b * 6 + 3 + c]);
    }
  const double qmax = (D == 3) ? double((1 << 21) - 1) : double((1u << 31) - 1);
  double sc[3];
  for (int c = 0; c < 3; ++c) sc[c] = (c < D && hi[c] > lo[c]) ? qmax / (hi[c] - lo[c]) : 0.0;
  uint64_t *keys = nullptr, *keys_out = nullptr;
  int32_t *idx = nullptr;
  FEM_CUDA(cudaMalloc(&keys, sizeof(uint64_t) * p->n_nodes));
  FEM_CUDA(cudaMalloc(&keys_out, sizeof(uint64_t) * p->n_nodes));
  FEM_CUDA(cudaMalloc(&idx, sizeof(int32_t) * p->n_nodes));
  FEM_CUDA(cudaMalloc(&p->node_order, sizeof(int32_t) * p->n_nodes));
  const double3 dlo = make_double3(lo[0], lo[1], lo[2]), dsc = make_double3(sc[0], sc[1], sc[2]);
  if (D == 3) k_node_morton<3><<<grid_for(p->n_nodes), kThreads, 0, s>>>(p->coords, p->n_nodes, dlo, dsc, keys, idx);
  else k_node_morton<2><<<grid_for(p->n_nodes), kThreads, 0, s>>>(p->coords, p->n_nodes, dlo, dsc, keys, idx);
  size_t bytes = 0;
  FEM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys_out, idx, p->node_order, (int)p->n_nodes, 0, 64, s));
  fem_status st = ensure(p->tmp, bytes);
  if (st) return st;
  FEM_CUDA(cub::DeviceRadixSort::SortPairs(p->tmp.ptr, bytes, keys, keys_out, idx, p->node_order, (int)p->n_nodes, 0, 64, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  cudaFree(keys); cudaFree(keys_out); cudaFree(idx);
  return FEM_OK;
}

void free_tiles(TileSet &T) {
  void *bufs[] = {T.perm, T.nodes, T.U, T.ptr, T.inc, T.lconn, T.interior, T.phase, T.slot_off,
                  T.node_slots, T.node_slot_ptr, T.epart, T.meta, T.list, T.geom, T.tcolor_list, T.refm, T.p2perm, T.meta_g8, T.p2n};
  for (void *b : bufs)
    if (b) cudaFree(b);
  T = TileSet{};
}

}  // namespace fem
