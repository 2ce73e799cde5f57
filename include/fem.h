/*
 * fem.h — C ABI of libfem.so, the B200 (sm_100a) hot path of the globally
 * differentiated energy FEM of arXiv 2602.12365 ("tatva", PAPER.md).
 *
 * The library evaluates the discrete energy Psi_h(u) = sum_e sum_q psi(grad u_h^e) w_q detJ^e
 * (Eq. 2) over P1 triangles (2D) and P1 tetrahedra (3D) for the
 * linear-elastic and compressible neo-Hookean (form fixed by
 * DESIGN.md reading C1) densities, its gradient r = grad Psi (Eq. 1), the
 * Hessian-vector product K(u) v (Eq. 3, §2.1), the sparsity pattern of K
 * (App. B), the distance-2 greedy coloring of its columns (§2.2,
 * P:184; App. A), the sparse tangent by Alg. 2 (one colored HVP per
 * color into J_comp, then decompression into CSR), SpMV, CG and Newton.
 * Derivatives are hand-derived per density (no AD framework).
 *
 * Conventions (all calls):
 *   - Array arguments are CUDA DEVICE pointers unless marked (host).  The caller owns
 *     every argument buffer (PyTorch tensors in the Python binding); the library owns
 *     its internal copies and workspaces and frees them in fem_destroy.  No call
 *     allocates caller-visible memory.
 *   - Values are fp64; node / element / DOF ids int32; CSR offsets int64.
 *   - DOF numbering: DOF = node * dim + comp (Alg. 1), the
 *     n_mpc Lagrange multipliers follow as DOFs N_u .. N_u + n_mpc - 1.
 *     N = N_u + n_mpc.
 *   - Every call enqueues its kernels on `stream` and returns without synchronizing,
 *     EXCEPT calls that return host values (fem_create, fem_query, fem_color,
 *     fem_cg_solve, fem_newton_solve, fem_check), which synchronize `stream`.
 *   - Errors: argument / shape errors return FEM_ERR_INVALID_ARG before any launch.
 *     Conditions found on the device (neo-Hookean J <= 0, too many colors) set a
 *     device error word; synchronous calls return it, asynchronous calls leave it
 *     for the next synchronous call or fem_check.  Output contents are undefined when
 *     the status is not FEM_OK.  fem_last_error() gives a message (thread-local).
 *   - There is no CPU fallback: every computation runs in this library's kernels.
 */
#ifndef FEM_B200_H
#define FEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fem_problem fem_problem; /* opaque, library-owned */
typedef void *fem_stream;               /* a cudaStream_t (0 = legacy default stream) */

typedef enum {
  FEM_OK = 0,
  FEM_ERR_INVALID_ARG = 1,
  FEM_ERR_DEGENERATE_ELEMENT = 2, /* detJ <= 1e-14 * (bbox diagonal)^d (reading C20)   */
  FEM_ERR_INVERTED_ELEMENT = 3,   /* neo-Hookean J = det F <= 0           */
  FEM_ERR_NONFINITE = 4,
  FEM_ERR_CG_BREAKDOWN = 5,       /* p^T A p <= 0                          */
  FEM_ERR_NOT_CONVERGED = 6,      /* iteration cap reached; report still filled         */
  FEM_ERR_TOO_MANY_COLORS = 7,    /* coloring needs more than FEM_MAX_COLORS colors     */
  FEM_ERR_OUT_OF_MEMORY = 8,
  FEM_ERR_CUDA = 9,
  FEM_ERR_NCCL = 10
} fem_status;

enum { FEM_TRI3 = 3, FEM_TET4 = 4 };
enum { FEM_LINEAR_ELASTIC = 0, FEM_NEO_HOOKEAN = 1 };
enum { FEM_MAX_COLORS = 256 };

/* flags */
enum {
  FEM_APPLY_BC = 1u,        /* Dirichlet by condensation on full-length vectors (P:389-400,
                               reading C12): residual r[D] = 0; HVP y = P_f K P_f v + P_D v;
                               CSR = that operator (1 on the D diagonal, 0 elsewhere in D
                               rows/cols), pattern unchanged.                            */
  FEM_DETERMINISTIC = 2u,   /* atomic-free fixed-order scatter (bitwise reproducible)    */
  FEM_ASSEMBLE_LITERAL = 4u,/* fem_assemble_csr: Alg. 2 as written — C sequential colored
                               HVP passes into J_comp [N][C], then decompression.        */
  FEM_BASELINE_SCATTER = 8u,/* residual / HVP: one thread per element with element-level
                               fp64 atomics instead of the element tiles — the baseline the
                               tile kernels are measured against.         */
  FEM_LOCAL_ONLY = 16u,     /* residual / HVP on a rank of a multi-GPU problem: skip the
                               halo add and return this rank's partial sums (DOF-wise
                               terms — f_ext, Dirichlet rows — on owned DOFs only, zero
                               elsewhere), so fem_halo_pack + exchange + fem_halo_combine
                               yields the global result.                                 */
  FEM_ASSEMBLE_JCOMP = 32u, /* fem_assemble_csr: all color passes in ONE element sweep
                               into J_comp [N][C] (atomics), then decompression.         */
  FEM_ASSEMBLE_ROWS = 64u,  /* fem_assemble_csr: row-pull form (no J_comp buffer).         */
  FEM_ASSEMBLE_SCATTER = 128u,/* fem_assemble_csr: element-Hessian scatter-add with fp64
                               atomics (the paper's comparison path), not Alg. 2 */
  FEM_LINEARIZED = 256u,    /* fem_hvp / CG op 0: the tangent at the state of the last
                               fem_linearize (its z; the z argument is not read for the
                               state) — Newton-Krylov applies K(z) thousands of times */
  FEM_STREAM_GEOM = 512u,   /* residual / HVP: read each element's reference geometry
                               (cofactor rows c_a = det J G_a and det J, 80 B per Tet4) from a
                               per-element stream built once, loaded per tile by one TMA bulk
                               copy — Alg. 1's per-batch gather of grad N and det J
                                — instead of recomputing it from the coordinates.
                               Not with FEM_DETERMINISTIC / BASELINE_SCATTER / LINEARIZED. */
  FEM_COLORED_SCATTER = 1024u,/* residual / HVP: elements colored so that no two elements of
                               a color share a node (greedy in tile order, setup); one pass
                               per color, each element adds its nodal vectors to the output
                               with plain loads / stores — conflict-free without atomics,
                               deterministic (fixed color order).                         */
  FEM_TILE_COLORED = 2048u, /* residual / HVP: the element tiles colored so that tiles of a
                               color share no node; one tile pass per color, in-tile sums as
                               usual, tile-boundary sums written with plain read-add-write
                               instead of fp64 atomics — the color-ordered conflict-free
                               scatter at tile granularity; deterministic.                */
  FEM_ASSEMBLE_COLORED = 4096u,/* fem_assemble_csr: Alg. 2 in fused form — one pass per node
                               color; each seed node's D colored columns are evaluated from
                               its incident elements and written straight to their CSR slots
                               (conflict-free plain stores), no J_comp.  No multipliers.   */
  FEM_REFERENCE_METRIC = 8192u /* residual / HVP (neo-Hookean): read the per-element
                               reference metric {mu vol G_a.G_b, 1/det J}, computed once per
                               problem (Alg. 1's precomputed grad N and det J),
                               instead of recomputing the reference geometry from the
                               coordinates in every call (the default).  56 B/tet more
                               reads, ~50 FP64 operations fewer per tet; same results up to
                               rounding order.  Not with FEM_DETERMINISTIC.               */
};

typedef struct {
  int dim;                       /* 2 (Tri3) or 3 (Tet4); dofs per node m = dim            */
  int64_t n_nodes, n_elems;
  const double *coords;          /* [n_nodes][dim] row-major                               */
  const int32_t *conn;           /* [n_elems][dim+1], positively oriented (detJ > 0)       */
  int material;                  /* FEM_LINEAR_ELASTIC or FEM_NEO_HOOKEAN                  */
  double lambda, mu;             /* uniform Lame parameters                        */
  const uint8_t *phase;          /* optional [n_elems] phase id (NULL = uniform)           */
  const double *lambda_tab;      /* (host) [n_phases] when phase != NULL                   */
  const double *mu_tab;          /* (host) [n_phases]                                      */
  int n_phases;
  int64_t n_dirichlet;
  const int32_t *dirichlet_dofs; /* [n_dirichlet] sorted, unique, < N_u                    */
  const double *dirichlet_vals;  /* [n_dirichlet] prescribed values g                      */
  int64_t n_mpc;                 /* g_k(u) = u[slave_k] - u[master_k] - offset_k */
  const int32_t *mpc_slave;      /* [n_mpc] < N_u                                          */
  const int32_t *mpc_master;     /* [n_mpc] < N_u, != slave_k                              */
  const double *mpc_offset;      /* [n_mpc]                                                */
  const double *f_ext;           /* optional [N_u] nodal load, Psi -= f_ext . u (NULL = 0) */
} fem_mesh_desc;

/* Element-partitioned multi-GPU run.  NULL => single GPU.
 * The mesh passed to fem_create is this rank's submesh (local node numbering in
 * ascending global id).  Interface nodes are listed per neighbour rank in ascending
 * global id; the halo add sums the partials of a shared DOF over the ranks touching it
 * in ascending rank order, so every rank holds the same bits. */
typedef struct {
  void *nccl_comm;               /* ncclComm_t from fem_nccl_comm_init                      */
  int rank, size;
  int n_nbr;
  const int32_t *nbr_rank;       /* (host) [n_nbr] ascending                               */
  const int64_t *nbr_offset;     /* (host) [n_nbr+1] offsets into nbr_nodes                */
  const int32_t *nbr_nodes;      /* (host) local node ids shared with each neighbour       */
  const uint8_t *owned;          /* (host) [n_nodes] 1 if this rank owns the node
                                    (lowest rank touching it); used for dots / energy      */
} fem_dist_desc;

/* Copies the mesh description into library-owned device buffers (the caller may free
 * its buffers once `stream` passes this point), validates it (ids in range, detJ >
 * eps_det -> FEM_ERR_DEGENERATE_ELEMENT, MPC pairs distinct), and prepares the element
 * tiles.  Synchronizes `stream`. */
fem_status fem_create(fem_problem **p, const fem_mesh_desc *d, const fem_dist_desc *dist,
                      fem_stream stream);
fem_status fem_destroy(fem_problem *p);

/* (host) N = N_u + n_mpc; nnz valid after fem_sparsity; n_colors after fem_color
 * (else -1).  Synchronizes nothing. */
fem_status fem_query(const fem_problem *p, int64_t *n_total, int64_t *nnz, int32_t *n_colors);

/* Returns (and clears) the device error word.  Synchronizes `stream`. */
fem_status fem_check(fem_problem *p, fem_stream stream);

/* z[D] = g: the lift of the reduced functional. */
fem_status fem_apply_dirichlet(fem_problem *p, double *z, fem_stream stream);

/* energy (device scalar) = Psi_h(u) + lambda . g(u) - f_ext . u  (Eq. 2, Alg. 1 P:112-147,
 * P:498).  Deterministic (fixed-order two-pass reduction). */
fem_status fem_energy(fem_problem *p, const double *z, double *energy, fem_stream stream);

/* r = grad L(z) [N] (Eq. 1; reverse-mode analogue P:154): per element f_a = vol P(H) G_a
 * scatter-added, + B^T lambda, r_lambda = B u - b, - f_ext; FEM_APPLY_BC: r[D] = 0. */
fem_status fem_residual(fem_problem *p, const double *z, double *r, unsigned flags,
                        fem_stream stream);

/* energy and residual in ONE element pass (value and gradient of Eq. 1-2):
 * *energy (device scalar, [1]) as fem_energy, r [N] as fem_residual with `flags`; all
 * pointers device memory owned by the caller; z and r must not alias (FEM_ERR_INVALID_ARG).
 * Inverted elements set the device error word (FEM_ERR_INVERTED_ELEMENT at the next
 * fem_check).  Multi-GPU problems and the FEM_DETERMINISTIC / FEM_BASELINE_SCATTER modes
 * run the two calls. */
fem_status fem_energy_residual(fem_problem *p, const double *z, double *energy, double *r,
                               unsigned flags, fem_stream stream);

/* y = K(z) v [N] (Eq. 3, §2.1), K the Hessian of the Lagrangian:
 * y_u = K_uu v_u + B^T v_lambda, y_lambda = B v_u; FEM_APPLY_BC: y = P_f K P_f v + P_D v.
 * v and y must not alias. */
fem_status fem_hvp(fem_problem *p, const double *z, const double *v, double *y, unsigned flags,
                   fem_stream stream);

/* Builds (once) the CSR pattern of K: (i,j) present iff DOFs i, j belong to nodes sharing
 * an element, full dim x dim node blocks, plus [[., B^T],[B, 0]] multiplier rows/cols
 * (App. B); columns ascending.  If row_ptr / col_idx are
 * non-NULL, copies the pattern into them ([N+1] int64 / [nnz] int32; query nnz first by
 * calling with NULLs, then fem_query). */
fem_status fem_sparsity(fem_problem *p, int64_t *row_ptr, int32_t *col_idx, fem_stream stream);

/* Distance-2 greedy coloring of the pattern's columns, ascending column order, smallest
 * free color (App. A; reading C9): bit-identical to the sequential
 * greedy.  Builds the pattern if needed.  colors [N] (may be NULL); *n_colors (host).
 * Synchronizes `stream`. */
fem_status fem_color(fem_problem *p, int32_t *colors, int32_t *n_colors, fem_stream stream);

/* vals [nnz] in fem_sparsity order = the sparse tangent K(z); the colored modes follow Alg. 2:
 * for each color c the HVP along the implicit seed e_c (e_j = [color_j == c]) gives
 * J_comp[:, c]; K_ij = J_comp[i, color_j] (decompression).  Modes (flags):
 *   FEM_ASSEMBLE_LITERAL: C sequential per-color passes into J_comp [N][C] (the paper's
 *            lax.scan), then a decompression kernel;
 *   FEM_ASSEMBLE_JCOMP: all color passes in ONE element sweep (the passes are
 *            independent), accumulating J_comp with atomics, then decompression;
 *   FEM_ASSEMBLE_COLORED: C/D node-color passes; every seed node's D columns K e_j are
 *            gathered from its incident elements and stored at their decompressed slots
 *            (Alg. 2 fused: compress and decompress in one step, no J_comp; the columns of
 *            one color never share a slot, so no atomics).  Each pass runs node tiles of 4
 *            seeds of the color with their element contexts in shared memory (fallback for
 *            meshes the tile plan rejects: a warp per seed over HBM context records);
 *   FEM_ASSEMBLE_ROWS: NOT Alg. 2: the row-owner gather form of the element-Hessian
 *            assembly (the sum of element Hessians, which
 *            Alg. 2 reproduces exactly).  Each node's D rows sum the tangent blocks
 *            K^e_nm of its incident elements and store them at the row's CSR slots; it reads
 *            neither the coloring nor a J_comp buffer, is atomic-free and bitwise
 *            reproducible.  Node tiles of 16 Morton-ordered nodes (8 when a node has more
 *            than 16 off-diagonal slots: unstructured meshes) evaluate their elements'
 *            tangent contexts in shared memory (no context records in HBM); the diagonal
 *            block is minus the row's off-diagonal sum (element rows sum to zero);
 *   FEM_ASSEMBLE_SCATTER: not Alg. 2 but the assembly the paper compares it with (Fig. 4
 *            right): dense element Hessians scatter-added into vals with fp64
 *            atomics (run-to-run rounding differences of the atomic order);
 *   default (no mode flag): FEM_ASSEMBLE_ROWS (the fastest on B200; bench.py reports the
 *            colored Alg. 2 modes next to it as colored_assembly_ms).
 * flags may add FEM_APPLY_BC.  Builds the pattern and (for the Alg. 2 modes) the coloring if
 * needed; synchronizes `stream` only on that first setup. */
fem_status fem_assemble_csr(fem_problem *p, const double *z, double *vals, unsigned flags,
                            fem_stream stream);

/* y = K_csr x (pattern of fem_sparsity, values `vals`); row-ordered accumulation.  Patterns
 * of full dim x dim node blocks (no multiplier columns) use a node-block kernel that reads
 * the node adjacency instead of col_idx (same values, same per-row order up to the lane
 * reduction); otherwise plain CSR. */
fem_status fem_spmv(fem_problem *p, const double *vals, const double *x, double *y,
                    fem_stream stream);

typedef struct {
  int op;           /* 0: masked HVP at z (matrix-free); 1: CSR `vals` (SpMV)       */
  double rtol, atol;/* stop when ||r||_2 <= max(rtol ||b||_2, atol)                        */
  int max_iter;
  int jacobi;       /* 1: Jacobi, 2: node-block (D x D) Jacobi (op 1 only; 2: one GPU)    */
  int check_every;  /* read the residual norm on the host every k iterations (>= 1)        */
  unsigned hvp_flags; /* op 0: extra fem_hvp flags (FEM_LINEARIZED)                         */
} fem_cg_opts;

typedef struct {
  int iters, converged;
  double res0, res;
} fem_cg_report;

/* Textbook CG on the BC-applied operator.  x: in x0, out solution.
 * b[D] and x0[D] should be 0 (condensed system).  Synchronizes `stream`. */
fem_status fem_cg_solve(fem_problem *p, const double *z, const double *vals, const double *b,
                        double *x, const fem_cg_opts *opts, fem_cg_report *report,
                        fem_stream stream);

/* Linearize the tangent at z (jax.linearize analogue): caches per element the deformed-
 * configuration metric form of the neo-Hookean tangent — cofactor rows of x + u, the two
 * state scalars (mu - lam ln J, lam scaled by 1 / (d! J det J(x+u))) and mu G_a.G_b vol —
 * 136 B per Tet4 in element-tile order (nothing for linear elasticity), so FEM_LINEARIZED
 * HVPs skip the geometry, the log and the reciprocals (cfg 3: 0.76 ms, HBM-bound at ~69 %
 * of the copy bandwidth, vs 0.94 ms recomputing).  fem_newton_solve linearizes at every
 * iterate for its matrix-free CG (FEM_NEWTON_RECOMPUTE=1: recompute instead). */
fem_status fem_linearize(fem_problem *p, const double *z, fem_stream stream);

/* MINRES (Paige & Saunders) on the same BC-applied operator, for the symmetric indefinite
 * saddle-point system of the MPC Lagrangian [[K, B^T], [B, 0]] (CG does not
 * apply).  opts as for CG (jacobi must be 0); report.res = true ||b - A x||_2.
 * Synchronizes `stream`. */
fem_status fem_minres_solve(fem_problem *p, const double *z, const double *vals, const double *b,
                            double *x, const fem_cg_opts *opts, fem_cg_report *report,
                            fem_stream stream);

/* Volume average of the first Piola-Kirchhoff stress (= the Cauchy stress for linear
 * elasticity), (1/|Omega|) sum_e vol_e P(H_e), the macroscopic stress of homogenization
 * (P:530-538): sigma (host) [dim*dim] row-major, volume (host) = |Omega|.  Fixed-order
 * reduction.  Synchronizes `stream`. */
fem_status fem_mean_stress(fem_problem *p, const double *z, double *sigma, double *volume,
                           fem_stream stream);

/* External loads of the total potential energy (listing P:380-386; SURVEY §8(f)
 * f3): Psi -= int_St t . u dGamma (traction on boundary facets: Line2 in 2D, Tri3 in 3D) and
 * Psi -= int b . u dOmega (uniform body force).  Linear in u and, with P1 shape functions
 * and loads constant per facet, exactly the consistent nodal loads t |facet| / dim and
 * b vol / (dim+1): both are ADDED to the problem's f_ext (energy, residual and Newton use
 * it; the HVP is unchanged).  facets [n_facets][dim] node ids, traction [n_facets][dim]
 * (device).  On a multi-GPU problem every facet is passed to one rank (that of its element)
 * and the loads of shared nodes are summed over the ranks (halo add), so f_ext holds the
 * global nodal load on every rank.  Both synchronize `stream` (facet ids out of range:
 * INVALID_ARG).
 * fem_get_fext copies the accumulated f_ext [N_u] (device). */
fem_status fem_add_traction(fem_problem *p, int64_t n_facets, const int32_t *facets,
                            const double *traction, fem_stream stream);
fem_status fem_add_body_force(fem_problem *p, const double *b /* (host) [dim] */,
                              fem_stream stream);
fem_status fem_get_fext(fem_problem *p, double *f_ext, fem_stream stream);

typedef struct {
  double atol, rtol; /* outer: ||r|| <= max(atol, rtol ||r0||)                 */
  int max_iter;
  fem_cg_opts cg;    /* inner solve; cg.op 0 = Newton-Krylov, 1 = colored CSR      */
  double forcing;    /* inner tolerance of Newton step k (DESIGN reading R16):
                      *   0: eta_k = cg.rtol at every step (fixed; the default);
                      *   > 0: inexact Newton-Krylov with Eisenstat-Walker "choice 2" forcing
                      *   terms, gamma = forcing (in (0, 1]; 0.9 typical), alpha = 2:
                      *   eta_0 = 0.1, eta_k = min(0.1, gamma (||r_k|| / ||r_{k-1}||)^2),
                      *   safeguarded by gamma eta_{k-1}^2 when that exceeds 0.1, never
                      *   below cg.rtol, and at least 0.5 tau / ||r_k|| (tau = the outer
                      *   target) so the last step does not over-solve.  The converged z
                      *   satisfies the same outer test.  forcing > 1 or < 0: INVALID_ARG. */
} fem_newton_opts;

typedef struct {
  int iters, cg_iters, converged;
  double res0, res;
} fem_newton_report;

/* Full-step Newton on the condensed problem (Eq. 1): z starts at the lift; repeat
 * r = residual(z, BC); K(z) dz = -r by CG (MINRES when the problem has MPC multipliers);
 * z += dz.  Synchronizes `stream`. */
fem_status fem_newton_solve(fem_problem *p, double *z, const fem_newton_opts *opts,
                            fem_newton_report *report, fem_stream stream);

/* ---------------------------------------------------------------- virtual-work path (f4)
 * Non-variational problems by the principle of virtual work (§3.1): a
 * scalar field c on a P1 mesh with W(c, v) = sum_e vol_e [ D grad c . grad v + (w_e . grad c)
 * vbar_e ] + m sum_a V_a (c_a - cold_a) v_a (one-point rule: vbar_e = mean of v over the
 * element, w_e = mean nodal velocity; V_a = lumped nodal volume; m = 1/dt, 0 = steady) —
 * the advection-diffusion example of P:772-802 on a flat mesh.  r = grad_v W at v = 0
 * (P:232); the tangent K = grad_c r is non-symmetric (advection), applied matrix-free
 * (fem_vw_jvp) and solved with restarted GMRES.  Dirichlet nodes: r[D] = 0 and the masked
 * operator P_f K P_f + P_D, as for the elastic path. */
typedef struct fem_vw_problem fem_vw_problem; /* opaque, library-owned */
typedef struct {
  int dim;                          /* 2 (Tri3) or 3 (Tet4)                                   */
  int64_t n_nodes, n_elems;
  const double *coords;             /* [n_nodes][dim]                                         */
  const int32_t *conn;              /* [n_elems][dim+1], positively oriented                  */
  double diffusivity;               /* D >= 0                                                 */
  const double *velocity;           /* [n_nodes][dim] nodal velocity                          */
  double mass_coef;                 /* m = 1/dt >= 0 (lumped mass), 0: steady                 */
  int64_t n_dirichlet;
  const int32_t *dirichlet_nodes;   /* unique node ids                                        */
  const double *dirichlet_vals;
} fem_vw_desc;
typedef struct {
  int restart;                      /* Krylov dimension per cycle, 1..64                       */
  int max_iter;                     /* total Arnoldi steps                                    */
  double rtol, atol;                /* stop when ||b - A x|| <= max(rtol ||b||, atol)          */
} fem_gmres_opts;
/* create copies the inputs (host or device pointers); synchronizes `stream`. */
fem_status fem_vw_create(fem_vw_problem **p, const fem_vw_desc *d, fem_stream stream);
fem_status fem_vw_destroy(fem_vw_problem *p);
fem_status fem_vw_apply_dirichlet(fem_vw_problem *p, double *c, fem_stream stream);
/* r [n_nodes] = grad_v W(c, v)|_{v=0}; c_old may be NULL (= 0); flags: FEM_APPLY_BC */
fem_status fem_vw_residual(fem_vw_problem *p, const double *c, const double *c_old, double *r,
                           unsigned flags, fem_stream stream);
/* y = K x (FEM_APPLY_BC: the masked operator) */
fem_status fem_vw_jvp(fem_vw_problem *p, const double *x, double *y, unsigned flags,
                      fem_stream stream);
/* GMRES(restart) on the masked operator; x: in x0, out solution; report as for CG
 * (res = the Arnoldi residual estimate).  Synchronizes `stream`. */
fem_status fem_vw_gmres_solve(fem_vw_problem *p, const double *b, double *x,
                              const fem_gmres_opts *opts, fem_cg_report *report,
                              fem_stream stream);

/* NCCL bootstrap for fem_dist_desc: rank 0 creates the id, the caller
 * broadcasts its 128 bytes (torch.distributed), every rank initialises the comm. */
fem_status fem_nccl_unique_id(unsigned char id[128]);
fem_status fem_nccl_comm_init(const unsigned char id[128], int rank, int size, void **comm);
fem_status fem_nccl_comm_destroy(void *comm);
/* (host) number of ranks in the communicator (ncclCommCount); bench.py logs it. */
fem_status fem_nccl_comm_count(void *comm, int *count);

/* (host) n = 1 / 2 scalar all-reduce (sum) of a device buffer over the problem's ranks
 * (no-op on a single GPU); used for global dots in multi-GPU CG and the energy. */
fem_status fem_allreduce_sum(fem_problem *p, double *buf, int n, fem_stream stream);

/* Halo add in explicit steps (what fem_residual / fem_hvp / fem_spmv do internally with
 * NCCL on a multi-GPU problem; exposed so the exchange can be driven by another transport).
 * Buffers hold, per neighbour in ascending rank order, the shared nodes' dim values in
 * ascending global id (fem_dist_desc.nbr_offset segments); n_doubles = entries * dim.
 * combine: y[n] = sum over the ranks touching n in ascending rank order of their partials
 * (own y[n] or recvbuf), so every rank holds identical bits. */
fem_status fem_halo_size(const fem_problem *p, int64_t *n_doubles);
fem_status fem_halo_pack(fem_problem *p, const double *y, double *sendbuf, fem_stream stream);
fem_status fem_halo_combine(fem_problem *p, double *y, const double *recvbuf, fem_stream stream);

const char *fem_last_error(void);
const char *fem_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FEM_B200_H */
