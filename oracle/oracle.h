/*
 * oracle.h — twin ABI of the CPU oracle (fem_ref_*).  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load liboracle.so.  The product (libfem.so) never links,
 * includes or calls it, and this header is a hand-written copy of the argument
 * meanings in include/fem.h, not an #include of it.
 *
 * All pointers are HOST pointers.  fp64 values, int32 node/element/DOF ids,
 * int64 CSR offsets.  DOF = node*dim + comp, multipliers after
 * all displacement DOFs.  Return values are the status codes of fem.h
 * (0 OK, 1 invalid arg, 2 degenerate element, 3 inverted element, 4 non-finite,
 * 5 CG breakdown, 6 not converged, 8 out of memory).
 */
#ifndef FEM_ORACLE_H
#define FEM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int dim;                 /* 2 (Tri3) or 3 (Tet4); dofs per node m = dim        */
  int64_t n_nodes, n_elems;
  const double *coords;    /* [n_nodes][dim]                                      */
  const int32_t *conn;     /* [n_elems][dim+1]                                    */
  int material;            /* 0 linear elastic, 1 compressible neo-Hookean        */
  double lambda, mu;
  const uint8_t *phase;    /* optional [n_elems]; NULL = uniform                  */
  const double *lambda_tab, *mu_tab;
  int n_phases;
  int64_t n_dirichlet;
  const int32_t *dirichlet_dofs;  /* sorted unique, < N_u */
  const double *dirichlet_vals;
  int64_t n_mpc;
  const int32_t *mpc_slave, *mpc_master;
  const double *mpc_offset;
  const double *f_ext;     /* optional [N_u]; NULL = 0                             */
} fem_ref_mesh;

enum { FEM_REF_APPLY_BC = 1u };

int fem_ref_geometry(const fem_ref_mesh *m, double *G /*[E][dim+1][dim]*/, double *vol /*[E]*/);
int fem_ref_energy(const fem_ref_mesh *m, const double *z, double *energy);
int fem_ref_residual(const fem_ref_mesh *m, const double *z, double *r, unsigned flags);
int fem_ref_hvp(const fem_ref_mesh *m, const double *z, const double *v, double *y, unsigned flags);
int fem_ref_dense_hessian(const fem_ref_mesh *m, const double *z, double *H /*[N][N]*/, unsigned flags);
int fem_ref_residual_rows(const fem_ref_mesh *m, const double *z, int64_t n_rows, const int64_t *rows,
                          double *out, unsigned flags);
int fem_ref_hvp_rows(const fem_ref_mesh *m, const double *z, const double *v, int64_t n_rows,
                     const int64_t *rows, double *out, unsigned flags);
int fem_ref_sparsity(const fem_ref_mesh *m, int64_t *row_ptr /*[N+1]*/, int32_t *col_idx /*[nnz] or NULL*/);
int fem_ref_color(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, int32_t *colors,
                  int32_t *n_colors);
int fem_ref_assemble_alg2(const fem_ref_mesh *m, const double *z, const int64_t *row_ptr,
                          const int32_t *col_idx, const int32_t *colors, int32_t n_colors,
                          double *vals, unsigned flags);
int fem_ref_assemble_elem(const fem_ref_mesh *m, const double *z, const int64_t *row_ptr,
                          const int32_t *col_idx, double *vals, unsigned flags);
int fem_ref_csr_rows(const fem_ref_mesh *m, const double *z, const int64_t *row_ptr,
                     const int32_t *col_idx, int64_t n_rows, const int64_t *rows,
                     double *vals_out /* packed, row by row */, unsigned flags);
int fem_ref_spmv(int64_t n, const int64_t *row_ptr, const int32_t *col_idx, const double *vals,
                 const double *x, double *y);
/* op 0: masked HVP operator at z; op 1: CSR (row_ptr/col_idx/vals). */
int fem_ref_cg(const fem_ref_mesh *m, int op, const double *z, const int64_t *row_ptr,
               const int32_t *col_idx, const double *vals, const double *b, double *x,
               double rtol, double atol, int max_iter, int *iters, double *res0, double *res);
/* volume-averaged first Piola-Kirchhoff stress sigma[dim*dim] (row-major), *volume = |Omega| */
int fem_ref_mean_stress(const fem_ref_mesh *m, const double *z, double *sigma, double *volume);
/* consistent nodal loads (added into f[n_nodes*dim]) of a traction on facets [nf][dim]
 * (t [nf][dim]) and of a uniform body force b[dim] */
int fem_ref_traction_load(int dim, int64_t n_nodes, const double *coords, int64_t nf,
                          const int32_t *facets, const double *t, double *f);
int fem_ref_body_load(const fem_ref_mesh *m, const double *b, double *f);
/* virtual-work path (f4): scalar advection-diffusion on a P1 mesh */
typedef struct {
  int dim;
  int64_t n_nodes, n_elems;
  const double *coords;
  const int32_t *conn;
  double diffusivity;
  const double *velocity;   /* [n_nodes][dim] */
  double mass_coef;         /* 1/dt, lumped mass; 0 = steady */
  int64_t n_dirichlet;
  const int32_t *dirichlet_nodes;
  const double *dirichlet_vals;
} fem_ref_vw;
int fem_ref_vw_residual(const fem_ref_vw *p, const double *c, const double *cold, double *r,
                        unsigned flags);
int fem_ref_vw_jvp(const fem_ref_vw *p, const double *x, double *y, unsigned flags);
int fem_ref_newton(const fem_ref_mesh *m, double *z /* in: lift, out: solution */, double atol,
                   double rtol, int max_iter, double cg_rtol, int cg_max_iter, int *iters,
                   int *cg_iters_total, double *res0, double *res);

#ifdef __cplusplus
}
#endif
#endif
