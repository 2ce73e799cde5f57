// fem_internal.cuh — library-internal state and helpers of libfem.so (not installed).
//
// Data layout in HBM: coords [n_nodes][dim] fp64 AoS, conn [E][dim+1] int32
// (library copy, element order of the caller), node_bc [n_nodes] uint8 bit c = DOF
// node*dim+c is Dirichlet, CSR row_ptr int64 / col_idx int32, J_comp [N][C] fp64 row-major.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/fem.h"

// NVTX ranges around every C-ABI call (nsys / ncu --nvtx timelines); header-only NVTX v3,
// no-ops without an attached tool.  FEM_NVTX=0 compiles them out.
#ifndef FEM_NVTX
#define FEM_NVTX 1
#endif
#if FEM_NVTX
#include <nvtx3/nvToolsExt.h>
#endif

namespace fem {

#if FEM_NVTX
struct NvtxScope {
  explicit NvtxScope(const char *name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};
#define FEM_NVTX_RANGE(name) ::fem::NvtxScope fem_nvtx_scope_(name)
#else
#define FEM_NVTX_RANGE(name) \
  do {                       \
  } while (0)
#endif

enum : int { ERRW_INVERTED = 1, ERRW_TOO_MANY_COLORS = 2, ERRW_NONFINITE = 4, ERRW_ADJ_OVERFLOW = 8 };

constexpr int kMaxNodeAdj = 128;    // max distinct node neighbours (incl. self) per node (setup-time local arrays; Delaunay 3D meshes reach ~36)
constexpr int kRowMaxDeg = 256;     // max incident elements per node in the row-gather assembly fallback (k_rows_fused)
constexpr int kReduceBlocks = 1184; // 148 SMs x 8: fixed grid => fixed reduction order
constexpr int kThreads = 256;
#ifndef FEM_TILE
#define FEM_TILE 256
#endif
constexpr int kTile = FEM_TILE;     // elements per tile (one CTA)

enum { OP_ENERGY = 0, OP_RESIDUAL = 1, OP_HVP = 2, OP_HVP_LIN = 3, OP_LIN = 4, OP_RESIDUAL_S = 5,
       OP_HVP_S = 6, OP_RESIDUAL_R = 7, OP_HVP_R = 8 };
// OP_*_S: residual / HVP from the streamed per-element geometry (TileSet::geom; Alg. 1's
// per-batch gather of grad N and det J) instead of coordinates (FEM_STREAM_GEOM)
// OP_LIN: cache the tangent state at z (fem_linearize); OP_HVP_LIN: HVP from that cache
// OP_*_R: NH residual / HVP with the element's reference metric mu vol G_a.G_b and 1/det J
// read from TileSet::refm (mesh constants computed once, Alg. 1's precomputed grad N / det J,
// P:124-127) — only the deformed geometry at x + u is evaluated per call (FEM_REFERENCE_METRIC;
// A/B at cfg 3: HVP 0.986 vs 0.935 ms recomputed, residual 0.787 vs 0.805 ms — not the default)

// Element tiles (fem_tiles.cu).  maxe = kTile * (dim+1) reserved entries per tile.
struct TileSet {
  bool built = false;
  int64_t n_tiles = 0, n_slots = 0;
  // multi-GPU: tiles touching shared (interface) nodes first, then the interior tiles, so the
  // halo exchange overlaps the interior pass (fem_core.cu element_pass_halo)
  int32_t *list = nullptr;       // [n_tiles] boundary tiles, then interior tiles
  int64_t n_boundary = -1;       // -1: lists not built
  int maxe = 0, max_U = 0;
  int32_t *perm = nullptr;       // [E] tile order -> caller element id
  int32_t *nodes = nullptr;      // [n_tiles][maxe] sorted unique nodes (first U valid)
  int32_t *U = nullptr;          // [n_tiles]
  uint16_t *ptr = nullptr;       // [n_tiles][maxe+1] start of each node's incidences
  uint16_t *inc = nullptr;       // [n_tiles][maxe] packed (element_local << 2 | slot)
  uint16_t *lconn = nullptr;     // [n_tiles*kTile][4] tile-local node indices
  uint8_t *interior = nullptr;   // [n_tiles][maxe] all incident elements in the tile
  uint8_t *phase = nullptr;      // [E] permuted phase ids (if any)
  int64_t *slot_off = nullptr;   // [n_tiles+1] prefix sum of U (deterministic mode)
  int32_t *node_slots = nullptr; // [n_slots] slots of each node, tile order
  int64_t *node_slot_ptr = nullptr; // [n_nodes+1]
  double *epart = nullptr;       // [n_tiles] energy partials
  double *geom = nullptr;        // [n_tiles][D*D+1][kTile] cofactor rows c_a and det J (SoA per tile)
  double *refm = nullptr;        // [n_tiles][D(D+1)/2+1][kTile] mu vol G_a.G_b (a<=b, a,b>=1), 1/det J
  int32_t *tcolor_list = nullptr;  // FEM_TILE_COLORED: tiles of color c at [tcolor_off[c], ..)
  std::vector<int64_t> tcolor_off;
  // balanced phase-2 schedule (fem_tiles.cu k_build_sched): per tile sched_rounds x kTile
  // task slots {8 cb offsets (uint16), meta = r | n << 12 | pos << 16 | g << 20}
  int sched_rounds = 0;
  int me8 = 0;                   // G8: padded incidence entries per tile (multiple of 8)
  uint16_t *inc8 = nullptr, *ptr8 = nullptr;  // G8 staging for k_pack_meta
  uint16_t *soff = nullptr;      // [n_tiles][rounds*kTile][8]
  uint32_t *smeta = nullptr;     // [n_tiles][rounds*kTile]
  uint32_t *shdr = nullptr;      // [n_tiles] rounds | shuffle steps << 8
  // packed per-tile metadata blocks (fem_tiles.cu pack_tile_meta), mb bytes each
  uint8_t *meta = nullptr;
  int um = 0, mb = 0, off_nodes = 0, off_lconn = 0, off_ptr = 0, off_inc = 0, off_int = 0,
      off_bc = 0, off_ph = 0, off_soff = 0, off_smeta = 0, off_perm = 0;
  // second metadata layout for the HVP kernels (FEM_HVP_G8): incidence offsets in padded groups
  // of 8 (the G8 node sums); nodes / lconn / ptr at the default offsets
  uint8_t *meta_g8 = nullptr;
  int mb_g8 = 0, off_inc_g8 = 0, off_int_g8 = 0, off_bc_g8 = 0, off_ph_g8 = 0, off_perm_g8 = 0;
  uint16_t *p2perm = nullptr;    // [n_tiles][maxe] phase-2 thread -> tile node (FEM_P2_SORT) or task (FEM_P2_LSPLIT)
  int32_t *p2n = nullptr;        // [n_tiles] phase-2 task count (FEM_P2_LSPLIT)
  int pcap = 0;                  // phase-2 order / task entries per metadata block
};

// node-tile assembly plan (fem_rowtile.cu build_tile_plan)
struct RtPlan {
  int state = 0;                 // 0 not built, 1 built, -1 not eligible
  uint8_t *meta = nullptr;
  int64_t ntiles = 0;
  int layout[20] = {0};          // RtLayout fields
  int smem = 0;
  std::vector<int64_t> seg_tiles;  // first tile of each node-list segment (colors for ct)
};

struct Workspace {
  void *ptr = nullptr;
  size_t bytes = 0;
};

struct Problem {
  int dim = 0, nen = 0, material = 0;
  int64_t n_nodes = 0, n_elems = 0, n_u = 0, n_mpc = 0, N = 0, n_dir = 0;
  double lam = 0, mu = 0;
  int n_phases = 0;
  // mesh copies
  double *coords = nullptr;
  int32_t *conn = nullptr;
  uint8_t *phase = nullptr;
  double *lam_tab = nullptr, *mu_tab = nullptr;
  uint8_t *node_bc = nullptr;
  int32_t *dir_dofs = nullptr;
  double *dir_vals = nullptr;
  int32_t *mpc_s = nullptr, *mpc_m = nullptr;
  double *mpc_b = nullptr;
  double *f_ext = nullptr;
  // reductions
  double *partials = nullptr;   // [kReduceBlocks * 4]
  double *scal = nullptr;       // device scalars (CG etc.) [64]
  double *h_scal = nullptr;     // pinned host mirror [64]
  int *d_err = nullptr;
  // incidence (node -> (element, local node)), built with the pattern
  int64_t *inc_ptr = nullptr;   // [n_nodes+1]
  int32_t *inc = nullptr;       // [E*nen] packed e*nen+a, ascending e per node
  // node adjacency (sorted, incl. self)
  int64_t *nadj_ptr = nullptr;  // [n_nodes+1]
  int32_t *nadj = nullptr;
  // dof -> mpc constraint list
  int32_t *dmpc_ptr = nullptr;  // [n_u+1]
  int32_t *dmpc = nullptr;
  // CSR pattern
  bool have_pattern = false;
  int64_t nnz = 0;
  int64_t *row_ptr = nullptr;
  int32_t *col_idx = nullptr;
  int64_t *diag_pos = nullptr;  // [N] position of the diagonal in each row (-1 if absent)
  uint16_t *slot_list = nullptr; // fused assembly: per node (l << 2 | b) grouped by CSR slot
  uint16_t *slot_off = nullptr; // [nnz_node + n_nodes] slot offsets into each node's list
  int32_t *node_order = nullptr; // [n_nodes] Morton order of the nodes (assembly)
  // FEM_ASSEMBLE_COLORED: seed nodes grouped by node color (Morton order within a color) and
  // the transposed slot of each adjacency entry (fem_assemble.cu assemble_colored)
  int32_t *ncolor_list = nullptr;
  std::vector<int64_t> ncolor_off;
  uint8_t *tslot = nullptr;
  // row-pull assembly plan (fem_rows.cu build_row_plan), indexed by the position in
  // node_order; fixed strides es (block entries) and ss (off-diagonal slots + 1)
  int rp_state = 0;              // 0 not built, 1 built, -1 mesh not eligible (fallback)
  int rp_lpn = 0, rp_es = 0, rp_ss = 0;
  int32_t *epos = nullptr;       // [E] element -> record position (element tile order)
  int4 *rp_node = nullptr;       // {n, sno | sn<<8 | ds<<16 | bc(n)<<24, row_ptr[dim*n] lo, hi}
  uint32_t *rp_ent = nullptr;    // [n_pad*es] blocks (pos | a<<27 | b<<29) grouped by slot
  uint8_t *rp_soff = nullptr;    // [n_pad*ss] entry offsets of the off-diagonal slots
  uint8_t *rp_sbc = nullptr;     // [n_pad*ss] Dirichlet bits of each slot's node
  // fused node-tile assembly (fem_rowtile.cu): packed per-tile metadata blocks of the row
  // form (rt) and of the colored form on node-color tiles (ct)
  RtPlan rt, ct;
  // coloring
  bool have_colors = false;
  int32_t n_colors = -1;
  int32_t *colors = nullptr;    // [N]
  // workspaces
  Workspace jcomp, cgbuf, tmp, slotbuf, ctxbuf, nwbuf;  // nwbuf: Newton r, dz (+ CSR values)
  cudaStream_t cap_stream = nullptr;  // CUDA-graph capture of solver iterations
  int spmv_lpn = 0;             // node-block SpMV lanes per node (0 unset, -1 plain CSR)
  // element coloring for FEM_COLORED_SCATTER (fem_core.cu build_elem_colors): elements of
  // color c (caller ids, tile order) at ecolor_list[ecolor_off[c] .. ecolor_off[c+1])
  int32_t *ecolor_list = nullptr;
  std::vector<int64_t> ecolor_off;
  double *lin = nullptr;        // fem_linearize cache: [lin_words(D)][n_tiles*kTile] metric-form tangent, SoA
  bool lin_valid = false;
  TileSet tiles;
  // multi-GPU (fem_dist.cu)
  void *nccl = nullptr;
  int rank = 0, size = 1, n_nbr = 0;
  std::vector<int> nbr_rank_h;
  std::vector<int64_t> nbr_off_h;
  int64_t n_halo_entries = 0, n_halo_nodes = 0;
  int32_t *halo_send_nodes = nullptr, *halo_nodes = nullptr, *halo_src_ptr = nullptr,
          *halo_src = nullptr;
  double *sendbuf = nullptr, *recvbuf = nullptr;
  uint8_t *owned = nullptr;     // [n_nodes] (size > 1)
  uint8_t *shared = nullptr;    // [n_nodes] 1 if the node is on an interface (size > 1)
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_part_a = nullptr, ev_halo = nullptr;
};

// ------------------------------------------------------------------ error plumbing
void set_error(const std::string &msg);
fem_status cuda_status(cudaError_t e, const char *what);

#define FEM_CUDA(call)                                                     \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) return ::fem::cuda_status(e_, #call);           \
  } while (0)

#define FEM_LAUNCH_CHECK(what)                                             \
  do {                                                                     \
    cudaError_t e_ = cudaGetLastError();                                   \
    if (e_ != cudaSuccess) return ::fem::cuda_status(e_, what);            \
  } while (0)

#define FEM_ARG(cond, msg)                                                 \
  do {                                                                     \
    if (!(cond)) {                                                         \
      ::fem::set_error(msg);                                               \
      return FEM_ERR_INVALID_ARG;                                          \
    }                                                                      \
  } while (0)

fem_status ensure(Workspace &w, size_t bytes);
// Stream-ordered allocations from the device's default memory pool (cudaMallocAsync), which
// keeps up to kPoolKeep bytes of freed memory mapped for reuse: the setup paths (pattern,
// coloring) allocate and free GB-sized buffers per problem, and plain cudaMalloc / cudaFree
// map and unmap them every time (bench setup medians of fresh problems varied 14-52 ms).
// Memory from pool_alloc may be released with pool_free (stream-ordered) or cudaFree.
fem_status pool_alloc(void **ptr, size_t bytes, cudaStream_t s);
#define FEM_POOL(call)               \
  do {                               \
    fem_status fem_pool_st_ = (call); \
    if (fem_pool_st_) return fem_pool_st_; \
  } while (0)
void pool_free(void *ptr, cudaStream_t s);
fem_status read_error_word(Problem *p, cudaStream_t s);

inline int grid_for(int64_t n, int threads = kThreads, int max_blocks = 148 * 64) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

// ------------------------------------------------------------------ device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// Block sum of one value per thread; result valid in thread 0.  Fixed order.
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[BLOCK / 32];
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (lane < BLOCK / 32) ? sh[lane] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

// internal launchers shared between translation units
fem_status launch_dot(Problem *p, const double *a, const double *b, int64_t n, double *out,
                      cudaStream_t s);
fem_status build_pattern(Problem *p, cudaStream_t s);
fem_status build_colors(Problem *p, cudaStream_t s);
fem_status run_residual(Problem *p, const double *z, double *r, unsigned flags, cudaStream_t s);
fem_status run_residual_terms(Problem *p, const double *z, double *r, unsigned flags, cudaStream_t s);
fem_status run_hvp(Problem *p, const double *z, const double *v, double *y, unsigned flags,
                   cudaStream_t s);
fem_status run_spmv(Problem *p, const double *vals, const double *x, double *y, cudaStream_t s);
fem_status halo_add(Problem *p, double *y, cudaStream_t s);
fem_status build_tiles(Problem *p, cudaStream_t s);
// part: 0 all tiles, 1 the tiles touching interface nodes, 2 the other tiles (TileSet::list),
// 3 tile-colored passes with plain boundary writes (FEM_TILE_COLORED)
fem_status tile_pass(Problem *p, int op, const double *u, const double *v, double *out, bool mask,
                     bool det, double *partials, cudaStream_t s, int part = 0);
fem_status build_tile_lists(Problem *p, cudaStream_t s);
fem_status build_geom_stream(Problem *p, cudaStream_t s);                // fem_tiles.cu
fem_status build_refm(Problem *p, cudaStream_t s);                       // fem_tiles.cu
fem_status build_tile_colors(Problem *p, cudaStream_t s);                // fem_tiles.cu
fem_status halo_begin(Problem *p, const double *y, cudaStream_t s);
fem_status halo_end(Problem *p, double *y, cudaStream_t s);
void free_tiles(TileSet &T);
int tile_energy_partials(Problem *p, int op = OP_ENERGY);
// per-element tangent context records (k_elem_ctx, fem_assemble.cu): doubles per element
template <int D>
constexpr int ctx_stride() { return D == 3 ? 28 : 16; }  // [G_a g_a] a = 0..D, smu sc1 sc2, pad
fem_status morton_node_order(Problem *p, cudaStream_t s);
fem_status build_row_plan(Problem *p, cudaStream_t s);          // fem_rows.cu
fem_status launch_rows_pull(Problem *p, const double *ctx, double *vals, bool bc,
                             cudaStream_t s);
fem_status build_row_tiles(Problem *p, cudaStream_t s);                  // fem_rowtile.cu
fem_status run_linearize(Problem *p, const double *z, cudaStream_t s);   // fem_core.cu
fem_status launch_row_tiles(Problem *p, const double *z, double *vals, bool bc, cudaStream_t s);
fem_status build_colored_tiles(Problem *p, cudaStream_t s);              // fem_rowtile.cu
fem_status launch_colored_tiles(Problem *p, const double *z, double *vals, bool bc, cudaStream_t s);
fem_status dist_setup(Problem *p, const fem_dist_desc *d, cudaStream_t s);
void dist_free(Problem *p);
fem_status allreduce(Problem *p, double *buf, int n, cudaStream_t s);
__global__ void k_final_sum(const double *partials, int64_t n, double *out);

}  // namespace fem

struct fem_problem {
  fem::Problem p;
};
