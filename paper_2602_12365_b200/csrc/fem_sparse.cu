// fem_sparse.cu — sparsity pattern (a7) and distance-2 greedy coloring (a8).
//
// Pattern (App. B): node -> element incidence by a stable radix
// sort of the connectivity, per-node sorted neighbour sets (node adjacency incl. self),
// expansion into dim x dim DOF blocks with columns ascending, plus the multiplier rows and
// columns [[K, B^T], [B, 0]].  row_ptr int64 (nnz exceeds 2^31 at BASELINE cfg 4).
//
// Coloring (App. A; reading C9): the sequential ascending-order greedy is reproduced
// exactly by index-priority dataflow (Jones-Plassmann with priority = -index): a column is
// colored in the round after its last lower-indexed distance-2 neighbour was colored; at
// that moment the colored neighbours are exactly the lower-indexed ones, so the smallest
// free color equals the sequential choice.  Counters of uncolored lower neighbours are
// decremented by the coloring column; frontiers are compacted with atomics.  Without
// multipliers the DOF graph is the node graph with full dim x dim blocks, and the greedy
// on DOFs equals color(node*dim + c) = dim * C_node(node) + c (proof in DESIGN.md §6), so
// the node graph (dim^2 fewer distance-2 visits) is colored instead.
#include <cub/cub.cuh>

#include "fem_internal.cuh"

namespace fem {

// ------------------------------------------------------------------ incidence
__global__ void k_iota_count(const int32_t *conn, int64_t n, int32_t *idx, int64_t *cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    idx[i] = (int32_t)i;
    atomicAdd(reinterpret_cast<unsigned long long *>(cnt + conn[i]), 1ull);
  }
}

// sorted unique neighbour nodes of node n (incl. itself); returns count or -1 on overflow
__device__ int node_neighbours(const int64_t *inc_ptr, const int32_t *inc, const int32_t *conn,
                               int nen, int32_t n, int32_t *nb) {
  int cnt = 0;
  for (int64_t t = inc_ptr[n]; t < inc_ptr[n + 1]; ++t) {
    const int64_t e = inc[t] / nen;
    for (int b = 0; b < nen; ++b) {
      const int32_t c = conn[e * nen + b];
      int lo = 0, hi = cnt;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (nb[mid] < c) lo = mid + 1; else hi = mid;
      }
      if (lo < cnt && nb[lo] == c) continue;
      if (cnt == kMaxNodeAdj) return -1;
      for (int q = cnt; q > lo; --q) nb[q] = nb[q - 1];
      nb[lo] = c;
      ++cnt;
    }
  }
  return cnt;
}

__global__ void k_nadj_count(const int64_t *inc_ptr, const int32_t *inc, const int32_t *conn,
                             int nen, int64_t n_nodes, int64_t *cnt, int *err) {
  int32_t nb[kMaxNodeAdj];
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int c = node_neighbours(inc_ptr, inc, conn, nen, (int32_t)n, nb);
    if (c < 0) { atomicOr(err, ERRW_ADJ_OVERFLOW); cnt[n] = 0; }
    else cnt[n] = c;
  }
}

__global__ void k_nadj_fill(const int64_t *inc_ptr, const int32_t *inc, const int32_t *conn,
                            int nen, int64_t n_nodes, const int64_t *nadj_ptr, int32_t *nadj) {
  int32_t nb[kMaxNodeAdj];
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < n_nodes;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int c = node_neighbours(inc_ptr, inc, conn, nen, (int32_t)n, nb);
    for (int q = 0; q < c; ++q) nadj[nadj_ptr[n] + q] = nb[q];
  }
}

// dof -> constraint lists
__global__ void k_dmpc_count(const int32_t *s, const int32_t *m, int64_t nc, int32_t *cnt) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nc;
       k += (int64_t)gridDim.x * blockDim.x) {
    atomicAdd(cnt + s[k], 1);
    atomicAdd(cnt + m[k], 1);
  }
}

__global__ void k_dmpc_fill(const int32_t *s, const int32_t *m, int64_t nc, const int32_t *ptr,
                            int32_t *cursor, int32_t *list) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nc;
       k += (int64_t)gridDim.x * blockDim.x) {
    list[ptr[s[k]] + atomicAdd(cursor + s[k], 1)] = (int32_t)k;
    list[ptr[m[k]] + atomicAdd(cursor + m[k], 1)] = (int32_t)k;
  }
}

__global__ void k_row_len(const int64_t *nadj_ptr, const int32_t *dmpc_ptr, int64_t n_u,
                          int64_t N, int dim, int64_t *len) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= N;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t l = 0;
    if (r < n_u) {
      const int64_t n = r / dim;
      l = (nadj_ptr[n + 1] - nadj_ptr[n]) * dim;
      if (dmpc_ptr) l += dmpc_ptr[r + 1] - dmpc_ptr[r];
    } else if (r < N) {
      l = 2;
    }
    len[r] = l;
  }
}

__global__ void k_row_fill(const int64_t *nadj_ptr, const int32_t *nadj, const int32_t *dmpc_ptr,
                           const int32_t *dmpc, const int32_t *ms, const int32_t *mm, int64_t n_u,
                           int64_t N, int dim, const int64_t *row_ptr, int32_t *col_idx,
                           int64_t *diag_pos) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = row_ptr[r];
    if (r < n_u) {
      const int64_t n = r / dim;
      int64_t dpos = -1;
      for (int64_t t = nadj_ptr[n]; t < nadj_ptr[n + 1]; ++t) {
        const int32_t nb = nadj[t];
        if (nb == n) dpos = p + (r % dim);
        for (int c = 0; c < dim; ++c) col_idx[p++] = nb * dim + c;
      }
      diag_pos[r] = dpos;
      if (dmpc_ptr) {
        const int32_t lo = dmpc_ptr[r], hi = dmpc_ptr[r + 1];
        // ascending constraint ids (tiny lists: insertion sort while writing)
        for (int32_t q = lo; q < hi; ++q) {
          int32_t k = dmpc[q];
          int64_t w = p + (q - lo);
          col_idx[w] = (int32_t)(n_u + k);
          while (w > p && col_idx[w - 1] > col_idx[w]) {
            const int32_t t = col_idx[w - 1];
            col_idx[w - 1] = col_idx[w];
            col_idx[w] = t;
            --w;
          }
        }
      }
    } else {
      const int64_t k = r - n_u;
      const int32_t a = ms[k], b = mm[k];
      col_idx[p] = a < b ? a : b;
      col_idx[p + 1] = a < b ? b : a;
      diag_pos[r] = -1;
    }
  }
}

template <typename T>
static fem_status exclusive_scan(T *in, T *out, int64_t n, Workspace &tmp, cudaStream_t s) {
  size_t bytes = 0;
  FEM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
  fem_status st = ensure(tmp, bytes);
  if (st) return st;
  FEM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.ptr, bytes, in, out, n, s));
  return FEM_OK;
}

static fem_status build_incidence(Problem *p, cudaStream_t s) {
  const int64_t n = p->n_elems * p->nen;
  int32_t *idx = nullptr, *keys_out = nullptr;
  int64_t *cnt = nullptr;
  FEM_POOL(pool_alloc((void **)&p->inc_ptr, sizeof(int64_t) * (p->n_nodes + 1), s));
  FEM_POOL(pool_alloc((void **)&p->inc, sizeof(int32_t) * (n > 0 ? n : 1), s));
  FEM_POOL(pool_alloc((void **)&cnt, sizeof(int64_t) * (p->n_nodes + 1), s));
  FEM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (p->n_nodes + 1), s));
  if (n > 0) {
    FEM_POOL(pool_alloc((void **)&idx, sizeof(int32_t) * n, s));
    FEM_POOL(pool_alloc((void **)&keys_out, sizeof(int32_t) * n, s));
    k_iota_count<<<grid_for(n), kThreads, 0, s>>>(p->conn, n, idx, cnt);
    int bits = 1;
    while ((int64_t(1) << bits) < p->n_nodes) ++bits;
    size_t bytes = 0;
    FEM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, p->conn, keys_out, idx, p->inc,
                                             (int)n, 0, bits, s));
    fem_status st = ensure(p->tmp, bytes);
    if (st) return st;
    FEM_CUDA(cub::DeviceRadixSort::SortPairs(p->tmp.ptr, bytes, p->conn, keys_out, idx, p->inc,
                                             (int)n, 0, bits, s));
  }
  fem_status st = exclusive_scan(cnt, p->inc_ptr, p->n_nodes + 1, p->tmp, s);
  FEM_CUDA(cudaStreamSynchronize(s));
  pool_free(idx, s);
  pool_free(keys_out, s);
  pool_free(cnt, s);
  return st;
}

fem_status build_pattern(Problem *p, cudaStream_t s) {
  if (p->have_pattern) return FEM_OK;
  fem_status st = build_incidence(p, s);
  if (st) return st;
  // node adjacency
  int64_t *cnt = nullptr;
  FEM_POOL(pool_alloc((void **)&cnt, sizeof(int64_t) * (p->n_nodes + 1), s));
  FEM_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (p->n_nodes + 1), s));
  k_nadj_count<<<grid_for(p->n_nodes, 128), 128, 0, s>>>(p->inc_ptr, p->inc, p->conn, p->nen,
                                                          p->n_nodes, cnt, p->d_err);
  FEM_POOL(pool_alloc((void **)&p->nadj_ptr, sizeof(int64_t) * (p->n_nodes + 1), s));
  st = exclusive_scan(cnt, p->nadj_ptr, p->n_nodes + 1, p->tmp, s);
  if (st) return st;
  int64_t total = 0;
  FEM_CUDA(cudaMemcpyAsync(&total, p->nadj_ptr + p->n_nodes, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  st = read_error_word(p, s);
  if (st) { pool_free(cnt, s); return st; }
  FEM_POOL(pool_alloc((void **)&p->nadj, sizeof(int32_t) * (total > 0 ? total : 1), s));
  k_nadj_fill<<<grid_for(p->n_nodes, 128), 128, 0, s>>>(p->inc_ptr, p->inc, p->conn, p->nen,
                                                         p->n_nodes, p->nadj_ptr, p->nadj);
  // dof -> constraint lists
  if (p->n_mpc) {
    int32_t *dcnt = nullptr, *cursor = nullptr;
    FEM_POOL(pool_alloc((void **)&dcnt, sizeof(int32_t) * (p->n_u + 1), s));
    FEM_POOL(pool_alloc((void **)&cursor, sizeof(int32_t) * (p->n_u + 1), s));
    FEM_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(int32_t) * (p->n_u + 1), s));
    FEM_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int32_t) * (p->n_u + 1), s));
    FEM_POOL(pool_alloc((void **)&p->dmpc_ptr, sizeof(int32_t) * (p->n_u + 1), s));
    FEM_POOL(pool_alloc((void **)&p->dmpc, sizeof(int32_t) * 2 * p->n_mpc, s));
    k_dmpc_count<<<grid_for(p->n_mpc), kThreads, 0, s>>>(p->mpc_s, p->mpc_m, p->n_mpc, dcnt);
    st = exclusive_scan(dcnt, p->dmpc_ptr, p->n_u + 1, p->tmp, s);
    if (st) return st;
    k_dmpc_fill<<<grid_for(p->n_mpc), kThreads, 0, s>>>(p->mpc_s, p->mpc_m, p->n_mpc, p->dmpc_ptr,
                                                        cursor, p->dmpc);
    FEM_CUDA(cudaStreamSynchronize(s));
    pool_free(dcnt, s);
    pool_free(cursor, s);
  }
  // rows
  int64_t *len = nullptr;
  FEM_POOL(pool_alloc((void **)&len, sizeof(int64_t) * (p->N + 1), s));
  k_row_len<<<grid_for(p->N + 1), kThreads, 0, s>>>(p->nadj_ptr, p->dmpc_ptr, p->n_u, p->N,
                                                     p->dim, len);
  FEM_POOL(pool_alloc((void **)&p->row_ptr, sizeof(int64_t) * (p->N + 1), s));
  st = exclusive_scan(len, p->row_ptr, p->N + 1, p->tmp, s);
  if (st) return st;
  FEM_CUDA(cudaMemcpyAsync(&p->nnz, p->row_ptr + p->N, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  FEM_POOL(pool_alloc((void **)&p->col_idx, sizeof(int32_t) * (p->nnz > 0 ? p->nnz : 1), s));
  FEM_POOL(pool_alloc((void **)&p->diag_pos, sizeof(int64_t) * (p->N > 0 ? p->N : 1), s));
  k_row_fill<<<grid_for(p->N), kThreads, 0, s>>>(p->nadj_ptr, p->nadj, p->dmpc_ptr, p->dmpc,
                                                  p->mpc_s, p->mpc_m, p->n_u, p->N, p->dim,
                                                  p->row_ptr, p->col_idx, p->diag_pos);
  FEM_LAUNCH_CHECK("pattern fill");
  FEM_CUDA(cudaStreamSynchronize(s));
  pool_free(cnt, s);
  pool_free(len, s);
  p->have_pattern = true;
  return FEM_OK;
}

// ------------------------------------------------------------------ coloring
// Number of (r, k) paths with r in adj(j), k in adj(r), k < j (with multiplicity).
__global__ void k_color_init(const int64_t *gp, const int32_t *gi, int64_t nv, int32_t *cnt,
                             int32_t *colors) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nv;
       j += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = 0;
    for (int64_t p = gp[j]; p < gp[j + 1]; ++p) {
      const int32_t r = gi[p];
      for (int64_t q = gp[r]; q < gp[r + 1]; ++q) c += (gi[q] < j);
    }
    cnt[j] = c;
    colors[j] = -1;
  }
}

// Round t, phase 1: the frontier = uncolored vertices whose lower distance-2 neighbours are
// all colored (counter reached 0 in an earlier round), compacted with warp-aggregated atomics.
__global__ void k_color_select(const int32_t *cnt, const int32_t *colors, int64_t nv,
                               int32_t *frontier, int32_t *size) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j - threadIdx.x < nv;
       j += (int64_t)gridDim.x * blockDim.x) {
    const bool ready = j < nv && colors[j] < 0 && cnt[j] == 0;
    const unsigned mask = __ballot_sync(0xffffffffu, ready);
    if (!mask) continue;
    const int lane = threadIdx.x & 31, leader = __ffs(mask) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(size, __popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (ready) frontier[base + __popc(mask & ((1u << lane) - 1))] = (int32_t)j;
  }
}

// Round t, phase 2: one warp per frontier column j.  The lanes split j's rows r, collect
// the colors of the lower distance-2 neighbours in a per-lane bitmask, OR-reduce it across
// the warp, take the smallest free color (all lower neighbours are colored), then decrement
// the counters of the higher distance-2 neighbours with fire-and-forget reductions.
__global__ void __launch_bounds__(128) k_color_apply(const int64_t *gp, const int32_t *gi,
                                                     int32_t *cnt, int32_t *colors,
                                                     const int32_t *frontier, int32_t *sizes,
                                                     int slot, int32_t *done, int *err,
                                                     int32_t *max_color) {
  const int32_t n_cur = sizes[slot];
  if (blockIdx.x == 0 && threadIdx.x == 0) sizes[slot ^ 1] = 0;
  const int lane = threadIdx.x & 31;
  const int32_t warps = gridDim.x * (blockDim.x >> 5);
  for (int32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_cur; w += warps) {
    const int32_t j = frontier[w];
    const int64_t p0 = gp[j], p1 = gp[j + 1];
    uint32_t fb[FEM_MAX_COLORS / 32];
#pragma unroll
    for (int q = 0; q < FEM_MAX_COLORS / 32; ++q) fb[q] = 0u;
    for (int64_t p = p0 + lane; p < p1; p += 32) {
      const int32_t r = gi[p];
      for (int64_t q = gp[r]; q < gp[r + 1]; ++q) {
        const int32_t k = gi[q];
        if (k < j) {
          const int32_t c = colors[k];
          fb[c >> 5] |= 1u << (c & 31);
        }
      }
    }
    int32_t c = -1;
#pragma unroll
    for (int q = 0; q < FEM_MAX_COLORS / 32; ++q) {
      const uint32_t m = __reduce_or_sync(0xffffffffu, fb[q]);
      if (c < 0 && m != 0xffffffffu) c = q * 32 + __ffs(~m) - 1;
    }
    if (lane == 0) {
      if (c < 0) { atomicOr(err, ERRW_TOO_MANY_COLORS); c = FEM_MAX_COLORS - 1; }
      colors[j] = c;
      atomicMax(max_color, c);
      atomicAdd(done, 1);
    }
    for (int64_t p = p0 + lane; p < p1; p += 32) {
      const int32_t r = gi[p];
      for (int64_t q = gp[r]; q < gp[r + 1]; ++q) {
        const int32_t k = gi[q];
        if (k > j) atomicSub(cnt + k, 1);  // result unused: compiled to RED
      }
    }
  }
}

// Push form (FEM_COLOR_PUSH): the thread whose decrement brings a higher neighbour's counter
// to zero appends it to the next round's frontier, so no round rescans all vertices (the
// select kernel above reads cnt and colors of every vertex every round).  Frontiers alternate
// between two buffers; three size counters rotate (round t reads sizes[t % 3], appends to
// sizes[(t + 1) % 3] and clears sizes[(t + 2) % 3], which no kernel of round t touches).  Each
// counter reaches zero exactly once (decrements and the initial count use the same
// multiplicities), and the colors are the same as the sequential greedy's: a vertex is colored
// only after all its lower distance-2 neighbours, whatever the round.  Measured (r02, cfg 3,
// 10.3M DOFs, bit-exact 90 colors): 34.4 ms against 33.1 ms for select + apply — the rounds
// are bound by the distance-2 enumeration of the frontier, not by the scan; off.
#ifndef FEM_COLOR_PUSH
#define FEM_COLOR_PUSH 0
#endif
__global__ void __launch_bounds__(128) k_color_apply_push(const int64_t *gp, const int32_t *gi,
                                                          int32_t *cnt, int32_t *colors,
                                                          const int32_t *frontier, int32_t *next,
                                                          int32_t *sizes, int t3, int32_t *done,
                                                          int *err, int32_t *max_color) {
  const int32_t n_cur = sizes[t3];
  int32_t *n_next = sizes + (t3 + 1) % 3;
  if (blockIdx.x == 0 && threadIdx.x == 0) sizes[(t3 + 2) % 3] = 0;
  const int lane = threadIdx.x & 31;
  const int32_t warps = gridDim.x * (blockDim.x >> 5);
  for (int32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n_cur; w += warps) {
    const int32_t j = frontier[w];
    const int64_t p0 = gp[j], p1 = gp[j + 1];
    uint32_t fb[FEM_MAX_COLORS / 32];
#pragma unroll
    for (int q = 0; q < FEM_MAX_COLORS / 32; ++q) fb[q] = 0u;
    for (int64_t p = p0 + lane; p < p1; p += 32) {
      const int32_t r = gi[p];
      for (int64_t q = gp[r]; q < gp[r + 1]; ++q) {
        const int32_t k = gi[q];
        if (k < j) {
          const int32_t c = colors[k];
          fb[c >> 5] |= 1u << (c & 31);
        }
      }
    }
    int32_t c = -1;
#pragma unroll
    for (int q = 0; q < FEM_MAX_COLORS / 32; ++q) {
      const uint32_t m = __reduce_or_sync(0xffffffffu, fb[q]);
      if (c < 0 && m != 0xffffffffu) c = q * 32 + __ffs(~m) - 1;
    }
    if (lane == 0) {
      if (c < 0) { atomicOr(err, ERRW_TOO_MANY_COLORS); c = FEM_MAX_COLORS - 1; }
      colors[j] = c;
      atomicMax(max_color, c);
      atomicAdd(done, 1);
    }
    // the counters are decremented only after colors[j] is written: a vertex pushed by this
    // warp reads colors[j] in a later round (kernel boundary), so no fence is needed
    for (int64_t p = p0 + lane; p < p1; p += 32) {
      const int32_t r = gi[p];
      for (int64_t q = gp[r]; q < gp[r + 1]; ++q) {
        const int32_t k = gi[q];
        if (k > j && atomicSub(cnt + k, 1) == 1) next[atomicAdd(n_next, 1)] = k;
      }
    }
  }
}

__global__ void k_expand_node_colors(const int32_t *nc, int64_t n_nodes, int dim, int32_t *colors) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_nodes * dim;
       i += (int64_t)gridDim.x * blockDim.x)
    colors[i] = dim * nc[i / dim] + (int32_t)(i % dim);
}

// Colors the graph (gp, gi) with nv vertices into `colors`; returns the number of colors.
static fem_status greedy_color(Problem *p, const int64_t *gp, const int32_t *gi, int64_t nv,
                               int32_t *colors, int32_t *n_colors, cudaStream_t s) {
  int32_t *cnt = nullptr, *f0 = nullptr, *aux = nullptr;
  FEM_POOL(pool_alloc((void **)&cnt, sizeof(int32_t) * (nv > 0 ? nv : 1), s));
  // select form: one frontier; push form: two alternating frontiers
  FEM_POOL(pool_alloc((void **)&f0, sizeof(int32_t) * (FEM_COLOR_PUSH ? 2 : 1) * (nv > 0 ? nv : 1), s));
  FEM_POOL(pool_alloc((void **)&aux, sizeof(int32_t) * 8, s));  // sizes[2], done, max_color, push sizes[3]
  FEM_CUDA(cudaMemsetAsync(aux, 0, sizeof(int32_t) * 8, s));
  FEM_CUDA(cudaMemsetAsync(aux + 3, 0xff, sizeof(int32_t), s));  // max_color = -1
  int32_t *sizes = aux, *done = aux + 2, *maxc = aux + 3;
  k_color_init<<<grid_for(nv), kThreads, 0, s>>>(gp, gi, nv, cnt, colors);
  FEM_LAUNCH_CHECK("color init");
  int32_t h_done = 0;
  const int kCheck = 32;
  const int sel_grid = grid_for(nv, kThreads, 148 * 16);
  // push form: sizes[0..2] rotate (aux[0], aux[1], aux[4]); round 0's frontier by one select
  int32_t *psz = aux + 4;  // [3]
  if (FEM_COLOR_PUSH) {
    FEM_CUDA(cudaMemsetAsync(psz, 0, sizeof(int32_t) * 3, s));
    k_color_select<<<sel_grid, kThreads, 0, s>>>(cnt, colors, nv, f0, psz);
  }
  for (int t = 0; h_done < nv;) {
    for (int q = 0; q < kCheck; ++q, ++t) {
      if (FEM_COLOR_PUSH) {
        const int32_t *fin = f0 + (t & 1) * (nv > 0 ? nv : 1);
        int32_t *fout = f0 + ((t + 1) & 1) * (nv > 0 ? nv : 1);
        k_color_apply_push<<<148 * 4, 128, 0, s>>>(gp, gi, cnt, colors, fin, fout, psz, t % 3, done,
                                                   p->d_err, maxc);
      } else {
        const int slot = t & 1;
        k_color_select<<<sel_grid, kThreads, 0, s>>>(cnt, colors, nv, f0, sizes + slot);
        k_color_apply<<<148 * 4, 128, 0, s>>>(gp, gi, cnt, colors, f0, sizes, slot, done, p->d_err, maxc);
      }
    }
    FEM_LAUNCH_CHECK("color round");
    FEM_CUDA(cudaMemcpyAsync(&h_done, done, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    FEM_CUDA(cudaStreamSynchronize(s));
    if (t > 64 * (nv + 64)) {
      set_error("coloring did not terminate");
      return FEM_ERR_CUDA;
    }
  }
  int32_t hmax = -1;
  FEM_CUDA(cudaMemcpyAsync(&hmax, maxc, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FEM_CUDA(cudaStreamSynchronize(s));
  pool_free(cnt, s);
  pool_free(f0, s);
  pool_free(aux, s);
  *n_colors = hmax + 1;
  return read_error_word(p, s);
}

fem_status build_colors(Problem *p, cudaStream_t s) {
  if (p->have_colors) return FEM_OK;
  fem_status st = build_pattern(p, s);
  if (st) return st;
  FEM_POOL(pool_alloc((void **)&p->colors, sizeof(int32_t) * (p->N > 0 ? p->N : 1), s));
  int32_t nc = 0;
  if (p->n_mpc == 0) {
    int32_t *node_colors = nullptr;
    FEM_POOL(pool_alloc((void **)&node_colors, sizeof(int32_t) * p->n_nodes, s));
    st = greedy_color(p, p->nadj_ptr, p->nadj, p->n_nodes, node_colors, &nc, s);
    if (st) { pool_free(node_colors, s); return st; }
    if (nc * p->dim > FEM_MAX_COLORS) {
      pool_free(node_colors, s);
      set_error("coloring needs more than FEM_MAX_COLORS colors");
      return FEM_ERR_TOO_MANY_COLORS;
    }
    k_expand_node_colors<<<grid_for(p->n_u), kThreads, 0, s>>>(node_colors, p->n_nodes, p->dim,
                                                                p->colors);
    FEM_LAUNCH_CHECK("expand colors");
    FEM_CUDA(cudaStreamSynchronize(s));
    pool_free(node_colors, s);
    nc *= p->dim;
  } else {
    st = greedy_color(p, p->row_ptr, p->col_idx, p->N, p->colors, &nc, s);
    if (st) return st;
  }
  p->n_colors = nc;
  p->have_colors = true;
  return FEM_OK;
}

}  // namespace fem

using namespace fem;

extern "C" {

fem_status fem_sparsity(fem_problem *h, int64_t *row_ptr, int32_t *col_idx, fem_stream stream) {
  FEM_NVTX_RANGE("fem_sparsity");
  FEM_ARG(h, "fem_sparsity: null problem");
  Problem *p = &h->p;
  cudaStream_t s = (cudaStream_t)stream;
  fem_status st = build_pattern(p, s);
  if (st) return st;
  if (row_ptr)
    FEM_CUDA(cudaMemcpyAsync(row_ptr, p->row_ptr, sizeof(int64_t) * (p->N + 1), cudaMemcpyDeviceToDevice, s));
  if (col_idx && p->nnz)
    FEM_CUDA(cudaMemcpyAsync(col_idx, p->col_idx, sizeof(int32_t) * p->nnz, cudaMemcpyDeviceToDevice, s));
  return FEM_OK;
}

fem_status fem_color(fem_problem *h, int32_t *colors, int32_t *n_colors, fem_stream stream) {
  FEM_NVTX_RANGE("fem_color");
  FEM_ARG(h, "fem_color: null problem");
  Problem *p = &h->p;
  cudaStream_t s = (cudaStream_t)stream;
  fem_status st = build_colors(p, s);
  if (st) return st;
  if (colors)
    FEM_CUDA(cudaMemcpyAsync(colors, p->colors, sizeof(int32_t) * p->N, cudaMemcpyDeviceToDevice, s));
  if (n_colors) *n_colors = p->n_colors;
  FEM_CUDA(cudaStreamSynchronize(s));
  return FEM_OK;
}

}  // extern "C"
