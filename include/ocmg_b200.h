/*
 * ocmg_b200 -- C ABI of the B200-native all-at-once multigrid hot path.
 *
 * Drop-in boundary for the reference package `ocmg` (arXiv 1502.03917,
 * /root/reference/pkg/src/ocmg).  The reference's native seam is the numba
 * kernel pair in kernels.py, reached from smoothers.py; its other hot calls
 * are scipy CSR matvecs and a LAPACK LU.  Each entry point below replaces
 * one of those seams (reference file:line in the comment).  The Python shim
 * (paper_1502_03917_b200, ctypes) keeps the reference's class/function
 * names on top of this ABI.
 *
 * Conventions
 *   - plain C types only: int64_t sizes, double values, device pointers
 *     (e.g. torch.Tensor.data_ptr()) as `double*`, streams as `void*`
 *     (a cudaStream_t; NULL = legacy default stream);
 *   - every vector is fp64 in the reference's global dof layout
 *     (field-major, lexicographic inside a field; FieldLayout,
 *     assembly.py:205-226), so x / r / f tensors are interchangeable with the
 *     reference's numpy arrays after a host<->device copy;
 *   - calls are stream-ordered and asynchronous unless stated; a handle may
 *     be used by one stream at a time (SURVEY.md §8(b) threading row): a
 *     level owns device scratch (the exact-order sweep's progress flags and
 *     ring buffers, multicolour barriers, reduction partials), so two
 *     sweeps of the same level on different streams must be ordered by the
 *     caller with events, or they corrupt each other's scratch;
 *   - status: 0 ok; OCMG_E_ARG (-> ValueError), OCMG_E_CUDA
 *     (-> RuntimeError), OCMG_E_SINGULAR (-> SingularMatrixError,
 *     sparse.py:18-19); ocmg_last_error() returns the message of the last
 *     failure on the calling thread.
 */
#ifndef OCMG_B200_H
#define OCMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCMG_OK 0
#define OCMG_E_ARG (-1)
#define OCMG_E_CUDA (-2)
#define OCMG_E_SINGULAR (-3)
#define OCMG_E_STATE (-4)

/* problem ids */
#define OCMG_POISSON 0
#define OCMG_STOKES 1

/* smoother kinds (SmootherKind.name, smoothers.py:20) */
#define OCMG_SMOOTHER_NORMAL 0 /* NE-Jacobi  (reference "normal") */
#define OCMG_SMOOTHER_LSGS 1   /* NE-GS      (reference "lsgs")   */
#define OCMG_SMOOTHER_SLSGS 2  /* fwd + bwd NE-GS ("slsgs")        */
#define OCMG_SMOOTHER_CGS 3    /* collective GS over vertex pairs ("cgs") */
#define OCMG_SMOOTHER_VANKA 4  /* multiplicative patch smoother ("vanka"):
                                  forward pre-, backward post-smoothing */

/* NE-GS execution modes */
#define OCMG_GS_REFERENCE 0   /* level-scheduled, reference arithmetic (bitwise) */
#define OCMG_GS_WAVEFRONT 1   /* reference order, fused pipelined wavefront      */
#define OCMG_GS_MULTICOLOUR 2 /* distance-2 multicolour order (own convergence)  */

typedef struct ocmg_level ocmg_level;
typedef struct ocmg_transfer ocmg_transfer;
typedef struct ocmg_coarse ocmg_coarse;
typedef struct ocmg_hierarchy ocmg_hierarchy;

const char *ocmg_last_error(void);
int ocmg_abi_version(void);
int ocmg_device_sm_count(int *out);
/* total number of device kernels this library has launched (all threads);
 * differences around a region give the launches inside it. */
int ocmg_launch_count(int64_t *out);

/* ---- levels ----------------------------------------------------------- */

/* Generic level from a host CSR of the block operator A (canonical form:
 * sorted columns, no explicit zeros; SparseMatrix, sparse.py:30-58) and its
 * diagonal weight L (BlockSystem.norm_diag, assembly.py:230-257).
 * field_off: n_fields+1 offsets of the FieldLayout; pressure fields (Stokes)
 * are the ones flagged in pressure_mask (bit f = field f).
 * Precomputes what SmootherState.__init__ does (smoothers.py:189-216):
 * row_scaled = A_ij / L_j, n_diag_i = sum_j A_ij row_scaled_ij, the column
 * mirror, plus the NE-GS level schedule (both orders) and, when
 * want_colouring, a greedy distance-2 colouring. */
int ocmg_level_create_csr(int problem, int64_t n, const int64_t *row_off,
                          const int64_t *col, const double *val,
                          const double *norm_diag, int n_fields,
                          const int64_t *field_off, uint32_t pressure_mask,
                          int want_colouring, ocmg_level **out);

/* The control weight alpha of a generic (CSR) Poisson level: the collective
 * smoother's 2x2 solve divides by it (kernels.py:85-88), and it cannot be
 * recovered bitwise from the assembled -M/alpha block.  Structured levels
 * get it at creation. */
int ocmg_level_set_alpha(ocmg_level *lv, double alpha);

/* Structured P1 level (Poisson control, mesh level k >= 3): the operator is
 * held as position-class stencil tables (49 classes x 2 blocks x 7
 * offsets) built by the Python shim from the reference assembly rules
 * (assembly.py:97-131, 270-290), bit-identical to the assembled CSR.
 * tables: see ocmg_p1_tables layout in csrc/ocmg_p1.cuh (OCMG_P1_TABLE_DOUBLES
 * doubles). */
int ocmg_level_create_p1(int k, double alpha, const double *tables,
                         int64_t n_tables, ocmg_level **out);
int ocmg_level_destroy(ocmg_level *lv);
int64_t ocmg_level_n(const ocmg_level *lv);
/* analytic op count of one NE sweep (= nnz; kernels.py:25-39) */
int64_t ocmg_level_nnz(const ocmg_level *lv);

/* r = -(A x) + f   (BlockSystem.residual, assembly.py:259-263; f may be
 * NULL -> r = -(A x)). */
int ocmg_residual(const ocmg_level *lv, const double *x, const double *f,
                  double *r, void *stream);

/* One NE-Jacobi sweep (kernels.normal_sweep, kernels.py:17-39, via
 * normal_equation_sweep, smoothers.py:256-267): p = tau L^-1 A^T L^-1 r
 * from the entering r, x += p, r -= A p.  scratch: n doubles (the
 * reference's `update`, smoothers.py:206). *ops (optional, host) gets the
 * touched-entry count. */
int ocmg_ne_jacobi_sweep(const ocmg_level *lv, double tau, double *x,
                         double *r, double *scratch, void *stream,
                         int64_t *ops);

/* One NE-GS sweep (kernels.lsgs_sweep, kernels.py:43-66, via lsgs_sweep,
 * smoothers.py:270-278).  forward=1: index order; 0: reversed.
 * mode: OCMG_GS_* above. */
int ocmg_ne_gs_sweep(const ocmg_level *lv, int mode, int forward, double *x,
                     double *r, void *stream, int64_t *ops);

/* The same sweep with the residual out of place: reads r_in, leaves the new
 * residual in r_out (r_in may be overwritten).  This is the form the cycle
 * driver runs (ping-pong buffers, no copy-back) for the multicolour mode on
 * structured levels; other modes/levels copy r_in to r_out and sweep there.
 * Not a reference entry point: a B200 addition next to ocmg_ne_gs_sweep. */
int ocmg_ne_gs_sweep_into(const ocmg_level *lv, int mode, int forward, double *x,
                          double *r_in, double *r_out, void *stream,
                          int64_t *ops);

/* One multicolour NE-GS sweep of the rows [y_begin, y_end) of a structured
 * P1 level (a rank's strip).  x, r_in and r_out hold the
 * rows [slab_begin, slab_end) of both fields (field stride
 * (slab_end - slab_begin) * n1; a full-size vector is the slab [0, n1)),
 * with slab_begin <= max(0, y_begin - 29) and slab_end >= min(n1, y_end + 29);
 * the ghost rows of r_in must be current (the caller's halo exchange).  x is
 * updated in place on the strip's rows; r_out receives the strip's rows.
 * Strips tile the domain: the union of all ranks' sweeps is bit-identical to
 * ocmg_ne_gs_sweep(mode=MULTICOLOUR).  B200 addition (the reference is
 * single-process). */
int ocmg_ne_gs_sweep_strip(const ocmg_level *lv, int forward, int y_begin,
                           int y_end, int slab_begin, int slab_end, double *x,
                           const double *r_in, double *r_out, void *stream,
                           int64_t *ops);

/* Row-range forms for strip partitions (full-size vectors, only the rows
 * [begin, end) of the output computed; inputs need their ghost rows: one row
 * of x for the residual, one fine row for the restriction, one coarse row
 * for the prolongation).  Structured P1 levels/transfers only. */
int ocmg_residual_rows(const ocmg_level *lv, const double *x, const double *f,
                       double *r, int y_begin, int y_end, void *stream);
int ocmg_restrict_rows(const ocmg_transfer *t, const double *rf, double *rc,
                       int cy_begin, int cy_end, void *stream);
int ocmg_prolong_add_rows(const ocmg_transfer *t, const double *c, double *xf,
                          int fy_begin, int fy_end, void *stream);
/* The two halves of an NE-Jacobi sweep (kernels.normal_sweep, kernels.py:
 * 27-32 and 33-38) on the rows [y_begin, y_end) of a structured P1 level,
 * for a strip: p = tau W r / L needs r of rows y_begin-1 .. y_end; the apply
 * half (x += p, r -= A p) needs p of rows y_begin-1 .. y_end.  Full-size
 * vectors; the arithmetic of ocmg_ne_jacobi_sweep row for row. */
int ocmg_ne_jacobi_p_rows(const ocmg_level *lv, double tau, const double *r, double *p,
                          int y_begin, int y_end, void *stream);
int ocmg_ne_jacobi_apply_rows(const ocmg_level *lv, const double *p, double *x, double *r,
                              int y_begin, int y_end, void *stream);

/* One collective Gauss-Seidel sweep over state/adjoint vertex pairs
 * (kernels.collective_sweep, kernels.py:70-96, via cgs_sweep,
 * smoothers.py:288-295; Poisson control only): mode OCMG_GS_REFERENCE or
 * OCMG_GS_WAVEFRONT = the reference's vertex order (bit-identical),
 * OCMG_GS_MULTICOLOUR = 3-colour order (its own smoother).  scratch: n
 * doubles.  *ops: touched entries (nnz). */
int ocmg_cgs_sweep(const ocmg_level *lv, int mode, double *x, double *r,
                   double *scratch, void *stream, int64_t *ops);

/* Vanka patch smoother (SmootherState with kind "vanka", smoothers.py:87-176,
 * 205-209; Stokes only).  ocmg_level_set_vanka attaches the patches of a
 * generic (CSR) level -- the reference's build_vanka_patches output: patch
 * offsets (n_patches+1), global dof indices, and the local inverses padded
 * to mmax x mmax (row-major, mmax <= 32) -- and builds the dependency
 * schedule of the multiplicative sweep (patches whose dofs or residual
 * downdates share a row keep the reference's patch order).
 * ocmg_vanka_sweep is kernels.vanka_sweep (kernels.py:99-131) via
 * smoothers.vanka_sweep (smoothers.py:297-310): forward = patch order, else
 * reversed; bit-identical to the reference.  *ops: touched entries. */
int ocmg_level_set_vanka(ocmg_level *lv, int64_t n_patches, int mmax,
                         const int64_t *offsets, const int64_t *dofs,
                         const double *inverses);
int ocmg_vanka_sweep(const ocmg_level *lv, double tau, int forward, double *x,
                     double *r, void *stream, int64_t *ops);

/* Constant-mode removal of the pressure fields (pressure_mean_projection,
 * assembly.py:381-388); no-op for Poisson. */
int ocmg_mean_project(const ocmg_level *lv, double *x, void *stream);

/* out_dev[0] = sum_i w_i x_i^2 with w = L (BlockSystem.norm, squared,
 * assembly.py:265-267) when weighted, else sum x_i^2.  out_dev: device. */
int ocmg_norm2(const ocmg_level *lv, const double *x, int weighted,
               double *out_dev, void *stream);

/* ---- transfers (TransferPair, transfer.py:22-143) ---------------------- */

/* From the host CSR of the prolongation P (fine x coarse); R = P^T is built
 * on the device in canonical order (TransferPair.from_prolongation,
 * transfer.py:29-31). */
int ocmg_transfer_create_csr(int64_t nf, int64_t nc, const int64_t *row_off,
                             const int64_t *col, const double *val,
                             ocmg_transfer **out);
/* Structured block-P1 transfer (Poisson, both fields) level kc -> kc+1. */
int ocmg_transfer_create_p1(int kc, int n_fields, ocmg_transfer **out);
int ocmg_transfer_destroy(ocmg_transfer *t);
/* rc = R rf  (multigrid.py:148) */
int ocmg_restrict(const ocmg_transfer *t, const double *rf, double *rc,
                  void *stream);
/* xf += P c  (multigrid.py:153) */
int ocmg_prolong_add(const ocmg_transfer *t, const double *c, double *xf,
                     void *stream);

/* ---- coarse solve (CoarseSolver, multigrid.py:67-102) ------------------ */

/* lu/piv: LAPACK getrf output of the (pinned, for Stokes) dense coarsest
 * operator, column-major n x n, 0-based pivots.  For Stokes, p_off/mu_off
 * are the first dofs of the pressure fields, n_p their size (the pinned
 * dofs are p_off and mu_off); ignored for Poisson. */
int ocmg_coarse_create(int problem, int64_t n, const double *lu,
                       const int64_t *piv, int64_t p_off, int64_t mu_off,
                       int64_t n_p, ocmg_coarse **out);
int ocmg_coarse_destroy(ocmg_coarse *c);
int ocmg_coarse_solve(const ocmg_coarse *c, const double *rhs, double *x,
                      void *stream);

/* ---- hierarchy and cycle driver (Multigrid, multigrid.py:105-204) ------ */

typedef struct ocmg_cycle_config {
    int cycle_w;      /* 0: V-cycle, 1: W-cycle (CycleConfig.cycle) */
    int nu_pre;       /* CycleConfig.nu_pre */
    int nu_post;      /* CycleConfig.nu_post */
    int smoother;     /* OCMG_SMOOTHER_* */
    int gs_mode;      /* OCMG_GS_* */
    double tau;       /* NE-Jacobi damping (resolved_tau) */
} ocmg_cycle_config;

/* levels[0] is the coarsest smoothed level (hierarchy index 1); transfers[i]
 * connects hierarchy index i (coarse) and i+1 (fine); n_levels counts the
 * smoothed levels, so there are n_levels transfers (the first one from the
 * coarse-solve level).  Handles stay owned by the caller. */
int ocmg_hierarchy_create(int n_levels, ocmg_level *const *levels,
                          ocmg_transfer *const *transfers, ocmg_coarse *coarse,
                          const ocmg_cycle_config *cfg, ocmg_hierarchy **out);
int ocmg_hierarchy_destroy(ocmg_hierarchy *h);
/* One cycle on the finest level: x <- cycle(x, f) (multigrid.py:130-159)
 * followed by nothing else.  x, f: finest-level device vectors. */
int ocmg_cycle(ocmg_hierarchy *h, double *x, const double *f, void *stream);
/* The coarse correction of hierarchy index level_index (1..n_levels) for
 * the restricted residual crhs (its coarse level's length): corr = rec
 * cycles of index level_index - 1 from zero (rec = 2 for a W-cycle above
 * the coarse solve, multigrid.py:150-152).  Outside the reference mode the
 * library collapses that map for the coarse end of the hierarchy (levels of
 * at most 8450 unknowns below the finest) into one dense matrix built at
 * ocmg_hierarchy_create from the same device cycle on unit vectors; this
 * call applies whichever form the cycle uses (partitioned cycles call it to
 * stay bit-identical to ocmg_cycle). */
int ocmg_coarse_correction(ocmg_hierarchy *h, int level_index, const double *crhs,
                           double *corr, void *stream);
/* *level_index = the hierarchy index c whose visits the cycle has collapsed
 * into the coarse correction of index c + 1 (0: none). */
int ocmg_hierarchy_collapsed_level(const ocmg_hierarchy *h, int *level_index);
/* BASELINE protocol loop: repeat { cycle; mean projection; rel =
 * ||f-Ax||_2/||f||_2 } until rel <= tol or max_cycles.  hist (host,
 * max_cycles doubles) receives rel per cycle; *n_done the cycle count.
 * use_graph: capture one cycle in a CUDA graph and replay it. */
int ocmg_solve(ocmg_hierarchy *h, double *x, const double *f, double tol,
               int max_cycles, int use_graph, double *hist, int *n_done,
               void *stream);
/* ocmg_solve with the reference's divergence stop made explicit
 * (multigrid.py:26 DIVERGENCE_FACTOR = 1e6, multigrid.py:198-200): the loop
 * also ends, with *diverged = 1, once rel > divergence_factor * rel0 (rel0 =
 * the entering iterate's relative residual) or rel is not finite.
 * divergence_factor <= 0 disables the test.  ocmg_solve = this with 1e6. */
int ocmg_solve_ex(ocmg_hierarchy *h, double *x, const double *f, double tol,
                  int max_cycles, int use_graph, double divergence_factor,
                  double *hist, int *n_done, int *diverged, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* OCMG_B200_H */
