/*
 * sipref.h -- CPU ORACLE for PARSDMM (Peters & Herrmann, arXiv 1902.09699).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.
 * The product path (paper_1902_09699_b200/, include/sip.h) never links,
 * imports or calls anything in oracle/.  The two share no code, headers,
 * tables or helpers.
 *
 * Plain C99, fp64, single-threaded, no FMA contraction (-ffp-contract=off),
 * written to be checked against the paper by eye.  Citations "P:n" are
 * /root/reference/PAPER.md line numbers; "L<n>" are the readings of the
 * paper listed in DESIGN.md section 3 (SURVEY.md 8(c) ledger).
 *
 * Layout (reading L1): grids are (nz, ny, nx) row-major with x fastest,
 * m[(iz*ny + iy)*nx + ix]; 2D grids have ny = 1.  Operator outputs use the
 * COMPACT layouts of the paper: D_z x has (nz-1)*ny*nx entries, D_x x has
 * nz*ny*(nx-1), TV = [D_z; D_y; D_x] (D_y only in 3D), F x = (G x)[mask].
 */
#ifndef SIPREF_H
#define SIPREF_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { SIPREF_OP_I = 0, SIPREF_OP_DZ = 1, SIPREF_OP_DY = 2, SIPREF_OP_DX = 3,
       SIPREF_OP_TV = 4, SIPREF_OP_BLUR_MASK = 5 };
enum { SIPREF_BOUNDS = 0, SIPREF_L1 = 1, SIPREF_L2 = 2, SIPREF_ANNULUS = 3,
       SIPREF_CARD = 4, SIPREF_RANK = 5, SIPREF_NUCLEAR = 6, SIPREF_DCT_L1 = 7,
       SIPREF_HAAR_L1 = 8 };

typedef struct {
  int ndim;          /* 2 or 3 */
  int64_t n[3];      /* nz, ny, nx  (ny = 1 when ndim = 2) */
  double h[3];       /* hz, hy, hx */
} sipref_grid;

typedef struct {
  int op, type;
  double lo, hi;                 /* BOUNDS scalars                           */
  const double *lo_vec, *hi_vec; /* optional per-entry bounds, length M      */
  double sigma;                  /* L1 / L2 radius                           */
  double sigma_lo, sigma_hi;     /* ANNULUS                                  */
  int64_t k;                     /* CARD                                     */
  int relative;                  /* 1: sigma* are fractions of the norm of
                                    A m (l1 for L1, l2 for L2/ANNULUS) and
                                    k = floor(k_frac * M)  (reading L4, L23) */
  double k_frac;
  const double *kernel; int kh, kw;  /* BLUR_MASK: kh x kw kernel, row major */
  const unsigned char *mask;         /* BLUR_MASK: N bytes, 1 = observed     */
  int app_mode;      /* 0: the whole vector A m; 1: each x-fiber (row) of the
                        operator's grid-shaped output; 2: each z-fiber
                        (column) -- the projector is applied to every fiber
                        independently ("each row/column
                        independently"; NEXT-1).  Single-block operators.   */
  int64_t fib_len;   /* fiber length (set by sipref_fiber_len)               */
  sipref_grid tgrid; /* DCT_L1 / HAAR_L1: the grid of the transform (resolve) */
  int64_t mrows, mcols;  /* RANK / NUCLEAR: the operator's output viewed as
                        matrices of mrows x mcols (row-major runs of the
                        compact layout): 2D grids one matrix (z, x), 3D grids
                        one per z-plane (y, x) -- reading L29; set by
                        sipref_matrix_shape                                */
} sipref_set;

typedef struct {
  int max_iter, n_cg;
  double rho0, gamma0, eps_evol, eps_feas, eps_corr;
  int adapt_every, check_every, hist_s;
  double rho_ratio_cap, gamma_max;
  int eq25;        /* 1: CG stops by Eq. 25; 0: exactly n_cg iterations    */
  int fixed_work;  /* 1: stop test evaluated but never acted on            */
  double cg_tol_floor; /* floor of the Eq. 25 target (10*eps of the dtype)  */
} sipref_options;

typedef struct {
  int iterations, cg_total, converged, breakdown;
  double r_evol;
  /* optional per-iteration records (caller-allocated, may be NULL) */
  int *cg_per_iter;     /* [max_iter]                                      */
  int *branch;          /* [max_iter * (p+1)], Alg. 2 branch code or -1    */
  double *rho_trace;    /* [max_iter * (p+1)] rho after the iteration      */
  double *gamma_trace;  /* [max_iter * (p+1)]                              */
  double *r_feas_trace; /* [max_iter * p], NaN when not a check iteration  */
  double *r_evol_trace; /* [max_iter]                                      */
  uint64_t *supp_hash;  /* [max_iter * p] CARD sets: sum (mod 2^64) of
                           sipref_supp_key over the support {j : y_j != 0}
                           after iteration k; 0 for other sets            */
  /* final values (caller-allocated, may be NULL) */
  double *r_feas;       /* [p]   */
  double *rho, *gamma;  /* [p+1] */
} sipref_log;

void sipref_default_options(sipref_options *o);

/* orthonormal DCT-II of a grid field along every axis (y = D x) or its
   inverse (x = D^T y); NEXT-3's transform-domain l1 set, reading L30 */
void sipref_dct(const sipref_grid *g, int inverse, const double *x, double *y);
/* orthonormal full-depth Haar wavelet transform along every axis (every
   length a power of two), y = H x, or its inverse; the HAAR_L1 set */
void sipref_haar(const sipref_grid *g, int inverse, const double *x, double *y);

/* matrix view of an operator's output for RANK / NUCLEAR sets (reading
   L29): rows x cols of one matrix; the number of matrices is M / (rows cols) */
void sipref_matrix_shape(const sipref_grid *g, int op, int64_t *rows, int64_t *cols);
/* singular values of a rows x cols row-major matrix (one-sided Jacobi,
   descending); sv holds min(rows, cols) values */
void sipref_svd_values(int64_t rows, int64_t cols, const double *a, double *sv);

/* support fingerprint key of entry j (compact layout) of operator op's
   output: splitmix64(b N + grid index of the owning point), b the block of
   a TV stack.  A test instrument (per-iteration support comparison). */
uint64_t sipref_supp_key(const sipref_grid *g, int op, int64_t j);

/* number of grid points; M of an operator (compact) */
int64_t sipref_npts(const sipref_grid *g);
int64_t sipref_op_len(const sipref_grid *g, const sipref_set *s);
/* length of one fiber of the operator's output (app_mode 1: the x extent of
   the output field, nx - 1 for D_x; app_mode 2: its z extent, nz - 1 for
   D_z); 0 for app_mode 0 */
int64_t sipref_fiber_len(const sipref_grid *g, const sipref_set *s);

/* y = A x  and  x = A^T y  (compact layouts) */
void sipref_apply_A(const sipref_grid *g, const sipref_set *s, const double *x, double *y);
void sipref_apply_AT(const sipref_grid *g, const sipref_set *s, const double *y, double *x);

/* q = (sum_i rho_i A_i^T A_i + rho_{p+1} I) p,  Eq. 23 */
void sipref_apply_C(const sipref_grid *g, int p, const sipref_set *sets,
                    const double *rho, const double *pv, double *q);

/* Euclidean projection of w (length M) onto the simple set C_i, Table 1.
   The set's parameters must already be absolute (relative == 0). */
void sipref_project(const sipref_set *s, int64_t M, const double *w, double *y);

/* distance prox, Eq. 22 */
void sipref_prox_dist(int64_t N, const double *m, double rho, const double *w, double *y);

/* Warm-started CG on C x = b (Eq. 25 when eq25 != 0): returns iterations.
   tol_out receives the relative-residual target used. */
int sipref_cg(const sipref_grid *g, int p, const sipref_set *sets, const double *rho,
              const double *b, double *x, int n_cg, int eq25, double *tol_out,
              int *breakdown);

/* Algorithm 2 on explicit vectors for one set: returns the branch code
   (0 both, 1 alpha only, 2 beta only, 3 none) and writes rho/gamma. */
int sipref_adapt_rho_gamma(int64_t M, const double *v_hat, const double *v_hat0,
                           const double *v, const double *v0,
                           const double *s, const double *s0,
                           const double *y, const double *y0,
                           double rho, double eps_corr, double *rho_new,
                           double *gamma_new);

/* Eq. 26 feasibility error of s = A x for one set (absolute parameters) */
double sipref_feas(const sipref_set *s, int64_t M, const double *sv);

/* Algorithm 1.  x (length N) receives the result.
   init_x/init_y/init_v: optional warm start (NULL = reading L13 defaults:
   x = m, y_i = A_i m, v_i = 0).  init_y/init_v are arrays of p+1 pointers.
   init_rho/init_gamma: optional starting parameters (NULL = rho0/gamma0).
   out_y/out_v (optional, p+1 pointers) receive the final y_i, v_i.
   Returns 0 converged, 1 not converged, <0 error. */
int sipref_parsdmm(const sipref_grid *g, int p, const sipref_set *sets,
                   const sipref_options *o, const double *m, double *x,
                   const double *init_x, double *const *init_y, double *const *init_v,
                   const double *init_rho, const double *init_gamma,
                   double *const *out_y, double *const *out_v,
                   sipref_log *log);

/* Algorithm 4 (parallel Dykstra) -- the comparator of the
   paper's Fig. 1 experiment.  Weights rho_i =
   1/p; P_{V_i} for A_i = I is the set's projector, otherwise PARSDMM with
   that one set (the role of ARADMM in the paper: "the same update
   scheme"), options `inner`, started from v_i.  Relative parameters are
   resolved once from m.  Stops when ||x^k - x^{k-1}|| / ||x^k|| < tol or at
   max_outer.  Per outer iteration the log records the paper's counters
   (P:497-501): the largest CG count among the sub-problems, the number of
   l1-ball projections (the inner iterations of the l1 sub-problems), and
   Eq. 26 of x^k for every set. */
typedef struct {
  int iterations;
  int *cg_max;        /* [max_outer] */
  int *l1_proj;       /* [max_outer] */
  int *inner_iters;   /* [max_outer * p] */
  double *r_feas;     /* [max_outer * p] */
  double *r_evol;     /* [max_outer] */
} sipref_dykstra_log;
int sipref_dykstra(const sipref_grid *g, int p, const sipref_set *sets, const sipref_options *inner,
                   int max_outer, double tol, const double *m, double *x, sipref_dykstra_log *log);

/* Algorithm 3 (multilevel).  Level l grid is the fine grid coarsened
   (l-1) times by 2 (box mean + stride, reading L23); h doubles per level.
   logs: array of n_levels logs (index 0 = finest), may be NULL. */
int sipref_parsdmm_multilevel(const sipref_grid *g, int p, const sipref_set *sets,
                              const sipref_options *o, int n_levels,
                              const double *m, double *x, sipref_log *logs);

/* multilevel transfers (exposed for pins) */
void sipref_restrict(const sipref_grid *fine, const double *f, double *c);
/* prolongation of one operator's field from the coarse to the fine grid:
   every block interpolated on its own shape (reading L23) */
void sipref_prolong_field(const sipref_grid *coarse, const sipref_grid *fine, int op,
                          const double *c, double *f);
/* relative parameters resolved from m (readings L4, L23): L1 sigma =
   frac ||A m||_1, L2 sigma = frac ||A m||_2, ANNULUS bounds x ||A m||_2,
   CARD k = floor(k_frac M) (the fiber length for per-fiber sets) */
void sipref_resolve_set(const sipref_grid *g, const sipref_set *in, const double *m,
                        sipref_set *out);
void sipref_interp(int64_t cz, int64_t cy, int64_t cx, const double *c,
                   int64_t fz, int64_t fy, int64_t fx, double *f);

#ifdef __cplusplus
}
#endif
#endif
