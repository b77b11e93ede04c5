/*
 * sip.h -- C ABI of the B200-native PARSDMM hot path (arXiv 1902.09699,
 * Peters & Herrmann, "Algorithms and software for projections onto
 * intersections of convex and non-convex sets ...").
 *
 * The library projects a 2D/3D gridded model m onto the intersection of
 * constraint sets V_i = {x : A_i x in C_i} (Eq. 14) with
 * PARSDMM (Algorithm 1), adaptive rho/gamma (Algorithm 2,
 * P:319-359), the Eq. 25 CG stop, the Eq. 26-28 stop rule
 * and multilevel continuation (Algorithm 3).
 * Citations "P:n" are lines of the paper text; "L<n>" are the
 * readings of the paper listed in DESIGN.md section 3.
 *
 * Conventions
 *  - Every function returns sip_status: 0 = OK, < 0 error, > 0 warning.
 *    On error the grid keeps its previous state; sip_last_error() gives a
 *    message.  Nothing is thrown across the ABI.
 *  - Layout (reading L1): grids are (nz[, ny], nx) row-major with x fastest
 *    (z slowest), x[(iz*ny + iy)*nx + ix]; 2D grids have no y axis.
 *  - Vector arguments marked "host or device" may be either; the library
 *    inspects the pointer (cudaPointerGetAttributes).  Host buffers are
 *    copied on the grid's stream inside the call.  Device buffers must be
 *    on the grid's device.
 *  - Vectors in an operator's range (per-entry bounds, sip_apply_op output,
 *    sip_project_set input/output, sip_get_state) use the paper's COMPACT
 *    layouts: D_z x has (nz-1)*ny*nx entries, D_y x nz*(ny-1)*nx, D_x x
 *    nz*ny*(nx-1), TV = [D_z; D_y; D_x] (D_y only in 3D), F x =
 *    (G x)[mask] in index order.  Internally the library stores padded
 *    grid-shaped fields.
 *  - Ownership: the grid handle owns all solver state (y_i, v_i, Alg. 2
 *    snapshots, work vectors).  It is allocated lazily by the first
 *    sip_project and reused ("set-up phase is a one time cost").
 *    Arguments are never retained after a call returns, except the data
 *    sip_add_set copies.
 *  - Thread safety: a grid handle is not thread safe; callers serialise.
 *  - Precision (reading L20): SIP_F32 stores vectors in fp32 and
 *    accumulates every reduction and every scalar in fp64; SIP_F64 is fp64
 *    throughout.
 */
#ifndef SIP_H
#define SIP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int sip_status;
#define SIP_OK              0
#define SIP_NOT_CONVERGED   1   /* max_iter reached; x holds the last iterate */
#define SIP_ERR_ARG        -1   /* NULL pointer, bad enum, bad key                    */
#define SIP_ERR_CONFIG     -2   /* operator unsupported for ndim, > 16 sets, ...      */
#define SIP_ERR_PARAM      -3   /* lo > hi, sigma < 0, sigma_lo > sigma_hi, bad k     */
#define SIP_ERR_SHAPE      -4   /* sizes inconsistent with the grid / operator        */
#define SIP_ERR_CUDA       -5
#define SIP_ERR_NCCL       -6
#define SIP_ERR_OOM        -7
#define SIP_ERR_NUMERIC    -8   /* NaN/Inf in the state                               */
#define SIP_ERR_STATE      -9   /* call out of order (e.g. get_state before project)  */

#define SIP_MAX_SETS 16         /* "up to about 16 sets"                      */

typedef struct sip_grid_s *sip_grid;

typedef enum { SIP_F32 = 0, SIP_F64 = 1 } sip_dtype;

/* Linear operators A_i (Table 1 rows use these) */
typedef enum {
  SIP_OP_IDENTITY = 0,  /* A = I                                            */
  SIP_OP_DZ = 1,        /* D_z (x) I: Eq. 8 forward difference along z / h_z */
  SIP_OP_DY = 2,        /* forward difference along y (3D only)              */
  SIP_OP_DX = 3,        /* forward difference along x                        */
  SIP_OP_TV = 4,        /* stacked [D_z; (D_y;) D_x]: one vector, one set    */
  SIP_OP_BLUR_MASK = 5  /* F = S G: G a 'same' zero-padded correlation with a
                           kh x kw kernel on the (z, x) plane, S keeps the
                           pixels where mask = 1 (2D grids, 1 rank only)     */
} sip_op;

/* Simple sets C_i, Table 1 */
typedef enum {
  SIP_SET_BOUNDS = 0,      /* lo <= (Ax)[i] <= hi, scalar or per entry      */
  SIP_SET_L1_BALL = 1,     /* ||Ax||_1 <= sigma                              */
  SIP_SET_L2_BALL = 2,     /* ||Ax||_2 <= sigma                              */
  SIP_SET_ANNULUS = 3,     /* sigma_lo <= ||Ax||_2 <= sigma_hi (non-convex)  */
  SIP_SET_CARDINALITY = 4, /* card(Ax) <= k (non-convex); ties: lowest index */
  SIP_SET_RANK = 5,        /* rank(A x as matrices) <= k (non-convex):
                              the truncated SVD of every matrix of the view
                              (reading L29: 2D grids one (z, x) matrix, 3D
                              grids one (y, x) matrix per z-plane); ties of
                              singular values: lowest index                   */
  SIP_SET_NUCLEAR = 6,     /* sum of singular values <= sigma per matrix of
                              the view; relative = 1: sigma is a
                              fraction of the summed nuclear norms of A m
                              (single-level projections only).  Both: single-
                              block operators, min(rows, cols) <= 2048, the
                              vectorised path (nx a multiple of 16 / sizeof),
                              one rank; else SIP_ERR_CONFIG                   */
  SIP_SET_DCT_L1 = 7,      /* ||D x||_1 <= sigma with D the orthonormal DCT-II
                              of the grid along every axis, kept inside the
                              set (P_V(x) = D^T P_l1(D x));
                              op must be IDENTITY; relative = 1: sigma is a
                              fraction of ||D m||_1 (reading L30); the
                              vectorised path, one rank (SIP_ERR_CONFIG)      */
  SIP_SET_HAAR_L1 = 8      /* ||H x||_1 <= sigma with H the orthonormal full-
                              depth Haar wavelet transform along every axis
                              (the paper's wavelet example, P:400-402;
                              reading L30); as DCT_L1, and every axis length
                              a power of two (else SIP_ERR_CONFIG)            */
} sip_set_type;

typedef struct {
  double lo, hi;          /* BOUNDS scalars, +-INFINITY allowed                 */
  const double *lo_vec;   /* optional per-entry bounds (host or device), length */
  const double *hi_vec;   /*   M of the operator, compact layout; copied at add */
  double sigma;           /* L1_BALL / L2_BALL radius >= 0                      */
  double sigma_lo, sigma_hi; /* ANNULUS, 0 <= lo <= hi                         */
  int64_t k;              /* CARDINALITY, 0 <= k <= M; RANK: the rank r >= 0   */
  double k_frac;          /* CARDINALITY with relative = 1: k = floor(k_frac*M) */
  int relative;           /* 1: sigma, sigma_lo, sigma_hi are fractions of the
                             norm of A m (l1 norm for L1_BALL, l2 otherwise),
                             re-derived from the m of every projection and every
                             multilevel level (readings L4, L23)               */
  int app_mode;           /* SIP_APPLY_*: the projector acts on the whole vector
                             A m (0), or on each x-fiber (row) / z-fiber
                             (column) of the operator's output field on its own
                             (NEXT-1): CARDINALITY (k per fiber; relative:
                             k = floor(k_frac * fiber length)), L1_BALL, L2_BALL
                             and ANNULUS (absolute radii per fiber; relative:
                             SIP_ERR_PARAM), single-block operators (not TV /
                             BLUR_MASK), fibers of <= 4096 entries, nx a
                             multiple of 16 / sizeof(dtype); on z slabs x-fibers
                             only.  BOUNDS accepts it (separable).  Else
                             SIP_ERR_CONFIG.                                    */
} sip_set_params;

enum { SIP_APPLY_WHOLE = 0, SIP_APPLY_X_FIBERS = 1, SIP_APPLY_Z_FIBERS = 2 };

typedef struct {
  const double *kernel;   /* host, kh*kw taps, row major (z rows, x columns)    */
  int kh, kw;             /* odd sizes, radius (kh/2, kw/2) <= 4                */
  const uint8_t *mask;    /* host or device, N bytes, 1 = observed pixel        */
} sip_blur_mask_desc;

typedef struct {
  int nranks, rank;              /* z-slab decomposition over nranks processes  */
  const uint8_t *nccl_unique_id; /* 128 bytes from sip_comm_unique_id on rank 0 */
} sip_comm_desc;

typedef struct {
  int iterations;       /* outer iterations k performed                         */
  int cg_iterations;    /* total CG iterations                                  */
  int converged;        /* Eq. 28 held at a check iteration                     */
  int breakdown;        /* CG met p.q <= 0                              */
  double r_evol;        /* Eq. 27 at the last check                             */
  double ms;            /* device time of the call (CUDA events)                */
  double r_feas[SIP_MAX_SETS];      /* Eq. 26 per set at the last check          */
  double rho[SIP_MAX_SETS + 1];     /* final rho_i, i = 1..p+1                   */
  double gamma[SIP_MAX_SETS + 1];   /* final gamma_i                             */
} sip_result;

/* ---- lifecycle ------------------------------------------------------- */

/* 128-byte NCCL unique id for a multi-rank grid (rank 0 calls it, the caller
   broadcasts it, e.g. with torch.distributed).  NCCL (libnccl.so.2) is
   loaded at the first call; SIP_ERR_NCCL if it is missing. */
sip_status sip_comm_unique_id(uint8_t out[128]);

/* The z-slab rule: of nz planes split over nranks, rank
   owns [z0, z0 + nz_local); nz_local = nz / nranks, plus one for the first
   nz mod nranks ranks.  Host only, no device work.  SIP_ERR_ARG on nz < 1,
   nranks < 1, rank outside [0, nranks) or NULL outputs. */
sip_status sip_slab(int64_t nz, int nranks, int rank, int64_t *z0, int64_t *nz_local);

/* Create a grid (compgrid).
   ndim: 2 or 3.  n: ndim counts, z first (each >= 2).  h: ndim spacings > 0
   (NULL = all 1, reading L2).  comm: NULL for one GPU, else the z-slab
   decomposition: the rank owns planes [z0, z0+nz_local) with the first
   nz mod nranks ranks holding one extra plane; m/x passed to this rank are
   its local slab (n stays the GLOBAL counts).  Every rank must call with
   the same n, h, dtype, sets and options; creation runs ncclCommInitRank
   (collective).  A multi-rank grid needs nx % (16 / sizeof(dtype)) == 0, no
   blur/mask operator and a single level; each step's reductions and 1-plane
   halos are exchanged with grouped NCCL send/recv (SIP_ERR_NCCL on
   failure).  cuda_stream: the caller's cudaStream_t (NULL = legacy
   default stream); every call orders its work after the work already queued
   on it, runs on a library-owned non-blocking stream (capturable into CUDA
   graphs) and returns after completion.  The current CUDA device at the
   call is the grid's device. */
sip_status sip_create_grid(int ndim, const int64_t *n, const double *h, sip_dtype dtype,
                           const sip_comm_desc *comm, void *cuda_stream, sip_grid *out);

/* Add a set V_i = {x : A x in C} (set_definitions).  op_desc is a
   sip_blur_mask_desc* for SIP_OP_BLUR_MASK, else NULL.  set_id receives
   i-1 (0-based, in order of addition).  Errors: SIP_ERR_CONFIG (DY on a 2D
   grid, blur on 3D or multi-rank, more than SIP_MAX_SETS sets),
   SIP_ERR_PARAM (lo > hi, sigma < 0, sigma_lo > sigma_hi, k out of range). */
sip_status sip_add_set(sip_grid g, sip_op op, const void *op_desc, sip_set_type type,
                       const sip_set_params *params, int *set_id);

/* Options (PARSDMM_options).  Keys and defaults:
   "rho0" 1e-2, "gamma0" 1, "n_cg" 10 (cap, L11), "eq25" 1 (0 = exactly n_cg
   CG steps), "fixed_work" 0 (1 = stop test evaluated, never acted on),
   "eps_evol" (default 10*tol of sip_project), "eps_corr" 0.3,
   "adapt_every" 2, "check_every" 5, "rho_ratio_cap" 1e3
   (L16), "gamma_max" 2-1e-3 (L15), "cg_tol_floor" 10*eps(dtype) (L18),
   "warm_start" 0 (1 = start from the grid's x, y_i, v_i, rho_i, gamma_i of
   the previous call instead of reading L13), "graph_iters" 10 (iterations
   per captured CUDA graph; 0 = no graph), "profile" 0 (1 = per-kernel event
   timing, see sip_get_profile; adds one host sync per graph launch),
   "virtual_ranks" 1 (G > 1: run the z-slab decomposition of G ranks on this
   one device -- the same per-slab kernels, finalisers and exchange schedule
   as the NCCL path, with device copies for the transfers; m and x stay
   whole-grid arrays; sip_project and sip_project_multilevel (the levels
   nest: nz divisible by G 2^(L-1)); SIP_ERR_PARAM unless 1 <= G <= nz and
   integral).
   Unknown key: SIP_ERR_ARG. */
sip_status sip_set_option(sip_grid g, const char *key, double value);

/* Project m onto the intersection (Algorithm 1).  m (read only) and x are
   N-vectors (host or device, grid dtype, must not alias); x receives the
   result.  max_iter >= 1.  tol sets eps_feas (Eq. 28) and, unless the
   option "eps_evol" was set, eps_evol = 10*tol (P:246's 1e-3 / 1e-2 pair);
   tol <= 0 keeps the options' values.  res may be NULL.
   Returns SIP_OK, SIP_NOT_CONVERGED, or an error. */
sip_status sip_project(sip_grid g, const void *m, void *x, int max_iter, double tol,
                       sip_result *res);

/* Multilevel PARSDMM (Algorithm 3): n_levels >= 1 levels, coarsening factor
   2 per axis (coarsen must be 2); every axis count must stay even down to
   the coarsest level.  Coarse m by 2x2(x2) block mean; x, y_i
   and v_i are prolonged by (tri)linear align-corners interpolation of each
   field as an image of its own shape; rho, gamma carry over.
   max_iter applies per level.  per_level (may be NULL) receives n_levels
   results, index 0 = finest.  On z slabs (NCCL ranks or virtual ranks) the
   levels nest when nz is divisible by G 2^(n_levels-1): restriction is
   slab-local, prolongation reads one coarse ghost plane per side after a
   halo exchange.  Not available for BLUR_MASK sets, per-entry bounds or a
   relative nuclear-norm radius (SIP_ERR_CONFIG). */
sip_status sip_project_multilevel(sip_grid g, const void *m, void *x, int n_levels,
                                  int coarsen, int max_iter, double tol,
                                  sip_result *per_level);

void sip_destroy(sip_grid g);
const char *sip_status_string(sip_status s);
const char *sip_last_error(sip_grid g);

/* ---- step-level entry points (the same device code as sip_project; used
        by the per-kernel parity tests) ---------------------------------- */

/* y = A_i x for set i: x an N-vector, y the compact M-vector (device or
   host, grid dtype). */
sip_status sip_apply_op(sip_grid g, int set_id, const void *x, void *y);

/* q = C p with C = sum_i rho_i A_i^T A_i + rho_{p+1} I (Eq. 23) for the
   given rho[0..p] (host array, p+1 entries); p, q N-vectors. */
sip_status sip_apply_system(sip_grid g, const double *rho, const void *p, void *q);

/* CG on C x = b (Eq. 23 with rho, host array of p+1), warm started at x
   (in/out).  eq25 = 1: stop rule Eq. 25; else exactly n_cg steps.
   iterations (may be NULL) receives the number of CG steps. */
sip_status sip_cg(sip_grid g, const double *rho, const void *b, void *x, int n_cg, int eq25,
                  int *iterations);

/* y = P_{C_i}(w) for set i (Table 1): w, y compact M-vectors.  Relative
   parameters are resolved against the m of the last projection (ERR_STATE
   if there was none). */
sip_status sip_project_set(sip_grid g, int set_id, const void *w, void *y);

/* Final y_i (which = 0) or v_i (which = 1) of the last projection in compact
   layout; set_id = p addresses the distance block y_{p+1}, v_{p+1}. */
sip_status sip_get_state(sip_grid g, int set_id, int which, void *out);

/* Per-iteration log of the last sip_project (host arrays, may be NULL):
   cg[max_iter] CG steps per iteration; branch[max_iter*(p+1)] Algorithm-2
   branch per set (0 both, 1 alpha only, 2 beta only, 3 none, -1 no adapt);
   rho_trace/gamma_trace[max_iter*(p+1)] after each iteration;
   r_feas[max_iter*p] and r_evol[max_iter] (NaN off check iterations). */
sip_status sip_get_log(sip_grid g, int max_iter, int *cg, int *branch, double *rho_trace,
                       double *gamma_trace, double *r_feas, double *r_evol);

/* Cardinality support fingerprints of the last sip_project run (a test
   instrument for SURVEY 8(c)'s "cardinality support at every iteration"):
   out[(k-1) * p + i] = sum mod 2^64 of splitmix64(b * N_global + global grid
   index of the owning point) over the non-zero entries of y_i after
   iteration k, b the operator block; 0 for sets that are not whole-vector
   cardinality sets.  Virtual ranks: summed over the slabs; NCCL ranks: this
   rank's slab only (sum over ranks to compare).  out holds max_iter * p
   uint64 (host).  Errors: SIP_ERR_ARG (null), SIP_ERR_STATE (no run). */
sip_status sip_get_support_log(sip_grid g, int max_iter, uint64_t *out);

/* Algorithm 4, parallel Dykstra: the comparator of the paper's
   Fig. 1 experiment.  Projects m onto the
   grid's sets with weights 1/p; P_{V_i} is the set's projector when its
   operator is IDENTITY, otherwise PARSDMM with that one set (natural mode,
   inner_max_iter iterations at most, tolerance inner_tol; the paper's
   ARADMM role), started from v_i.  Relative parameters are resolved
   once from m.  Stops when ||x^k - x^{k-1}|| / ||x^k|| < tol or after
   max_outer iterations (SIP_NOT_CONVERGED).  m, x: N-vectors (host or
   device).  log (host arrays, may be NULL): per outer iteration the largest
   CG count of the sub-problems, the l1-ball projections (inner iterations
   of the l1 sub-problems), inner iterations per set, Eq. 26 of x^k per set
   and r_evol.  One rank only (SIP_ERR_CONFIG). */
typedef struct {
  int iterations;
  int *cg_max;            /* [max_outer]     */
  int *l1_proj;           /* [max_outer]     */
  int *inner_iters;       /* [max_outer * p] */
  double *r_feas;         /* [max_outer * p] */
  double *r_evol;         /* [max_outer]     */
} sip_dykstra_log;
sip_status sip_dykstra(sip_grid g, const void *m, void *x, int max_outer, double tol, int inner_max_iter,
                       double inner_tol, sip_dykstra_log *log);

/* Number of sets p, grid points N (this rank) and compact length of set i. */
sip_status sip_get_sizes(sip_grid g, int *p, int64_t *n_local, int set_id, int64_t *m_compact);

/* Device time per kernel kind of the last sip_project run with option
   "profile" = 1 (CUDA event nodes between consecutive kernels, captured in
   the graph).  Kinds, in order: 0 blur (S G p), 1 rhs, 2 cg1, 3 cg2,
   4 pass1, 5 select, 6 tiecount, 7 pass2, 8 control, 9 comm (z-slab
   exchanges), 10 cgx (deferred CG x update), 11 fiber (per-fiber
   projections), 12 svd (rank / nuclear-norm sets), 13 dct (transforms of
   the transform-domain sets).  ms[q] is the summed milliseconds, count[q]
   the number of launches (arrays of n <= 14). */
sip_status sip_get_profile(sip_grid g, int n, double *ms, int64_t *count);

/* Number of kernel launches enqueued by the last sip_project (bench evidence). */
sip_status sip_get_launch_count(sip_grid g, int64_t *launches);

#ifdef __cplusplus
}
#endif
#endif
