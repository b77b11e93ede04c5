/*
 * sipref.c -- CPU ORACLE for PARSDMM (arXiv 1902.09699).  TEST INFRASTRUCTURE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
 * --impl reference arm) may load this code.  It shares nothing with the
 * CUDA product path.  Plain C99, fp64, single-threaded, compiled with
 * -O2 -ffp-contract=off (no FMA contraction, reading L20).
 *
 * Every function follows the paper in its own order and notation:
 *   operators    Eq. 8, TV stack, F = restriction of a
 *                blur (reading L21)
 *   projectors   Table 1; l1 by the sort of Duchi et al. 2008
 *                (P:501); distance prox Eq. 22
 *   system       Eq. 23: C = sum_i rho_i A_i^T A_i + rho_{p+1} I,
 *                applied literally set by set
 *   CG           warm start x^k, stop rule Eq. 25 (reading L18)
 *   PARSDMM      Algorithm 1 with Eq. 21
 *   adapt        Algorithm 2
 *   stopping     Eqs. 26-28
 *   multilevel   Algorithm 3, transfers per reading L23
 */
#include "sipref.h"
#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* small vector helpers (straight loops, index order)                  */
/* ------------------------------------------------------------------ */
static double dot(int64_t n, const double *a, const double *b) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
static double nrm2(int64_t n, const double *a) { return sqrt(dot(n, a, a)); }
static double *dalloc(int64_t n) {
  double *p = (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  return p;
}

void sipref_default_options(sipref_options *o) {
  o->max_iter = 200;      /* BASELINE.json C1, reading L11 */
  o->n_cg = 10;           /* "CG 10 inner iters" as a cap, L11 */
  o->rho0 = 1e-2;         /* BASELINE.json C1 */
  o->gamma0 = 1.0;
  o->eps_evol = 1e-2;
  o->eps_feas = 1e-3;
  o->eps_corr = 0.3;      /* Alg. 2 */
  o->adapt_every = 2;
  o->check_every = 5;     /* P:236 "typically 5" */
  o->hist_s = 5;          /* P:242 s = 5 */
  o->rho_ratio_cap = 1e3; /* reading L16 */
  o->gamma_max = 2.0 - 1e-3; /* reading L15 */
  o->eq25 = 1;
  o->fixed_work = 0;
  o->cg_tol_floor = 10.0 * DBL_EPSILON; /* reading L18 (fp32 runs: 10*FLT_EPSILON) */
}

/* ------------------------------------------------------------------ */
/* grid and operators                                                   */
/* ------------------------------------------------------------------ */
int64_t sipref_npts(const sipref_grid *g) { return g->n[0] * g->n[1] * g->n[2]; }

static int64_t IDX(const sipref_grid *g, int64_t iz, int64_t iy, int64_t ix) {
  return (iz * g->n[1] + iy) * g->n[2] + ix;
}

static int64_t len_dz(const sipref_grid *g) { return (g->n[0] - 1) * g->n[1] * g->n[2]; }
static int64_t len_dy(const sipref_grid *g) { return g->n[0] * (g->n[1] - 1) * g->n[2]; }
static int64_t len_dx(const sipref_grid *g) { return g->n[0] * g->n[1] * (g->n[2] - 1); }

static int64_t mask_count(const sipref_grid *g, const unsigned char *mask) {
  int64_t c = 0, N = sipref_npts(g);
  for (int64_t i = 0; i < N; ++i) c += mask[i] ? 1 : 0;
  return c;
}

int64_t sipref_op_len(const sipref_grid *g, const sipref_set *s) {
  switch (s->op) {
    case SIPREF_OP_I: return sipref_npts(g);
    case SIPREF_OP_DZ: return len_dz(g);
    case SIPREF_OP_DY: return g->ndim == 3 ? len_dy(g) : 0;
    case SIPREF_OP_DX: return len_dx(g);
    case SIPREF_OP_TV: return len_dz(g) + (g->ndim == 3 ? len_dy(g) : 0) + len_dx(g);
    case SIPREF_OP_BLUR_MASK: return mask_count(g, s->mask);
  }
  return 0;
}

/* Eq. 8: (D_z x)[iz,iy,ix] = (x[iz+1,iy,ix] - x[iz,iy,ix]) / h_z, iz < nz-1 */
static void dz_fwd(const sipref_grid *g, const double *x, double *y) {
  for (int64_t iz = 0; iz + 1 < g->n[0]; ++iz)
    for (int64_t iy = 0; iy < g->n[1]; ++iy)
      for (int64_t ix = 0; ix < g->n[2]; ++ix)
        y[(iz * g->n[1] + iy) * g->n[2] + ix] =
            (x[IDX(g, iz + 1, iy, ix)] - x[IDX(g, iz, iy, ix)]) / g->h[0];
}
/* transpose of Eq. 8: column iz of D_z^T has -1/h at row iz and +1/h at row iz-1 */
static void dz_adj(const sipref_grid *g, const double *y, double *x) {
  for (int64_t iz = 0; iz < g->n[0]; ++iz)
    for (int64_t iy = 0; iy < g->n[1]; ++iy)
      for (int64_t ix = 0; ix < g->n[2]; ++ix) {
        double a = 0.0;
        if (iz >= 1) a += y[((iz - 1) * g->n[1] + iy) * g->n[2] + ix];
        if (iz + 1 < g->n[0]) a -= y[(iz * g->n[1] + iy) * g->n[2] + ix];
        x[IDX(g, iz, iy, ix)] = a / g->h[0];
      }
}
static void dy_fwd(const sipref_grid *g, const double *x, double *y) {
  int64_t ny1 = g->n[1] - 1;
  for (int64_t iz = 0; iz < g->n[0]; ++iz)
    for (int64_t iy = 0; iy < ny1; ++iy)
      for (int64_t ix = 0; ix < g->n[2]; ++ix)
        y[(iz * ny1 + iy) * g->n[2] + ix] =
            (x[IDX(g, iz, iy + 1, ix)] - x[IDX(g, iz, iy, ix)]) / g->h[1];
}
static void dy_adj(const sipref_grid *g, const double *y, double *x) {
  int64_t ny1 = g->n[1] - 1;
  for (int64_t iz = 0; iz < g->n[0]; ++iz)
    for (int64_t iy = 0; iy < g->n[1]; ++iy)
      for (int64_t ix = 0; ix < g->n[2]; ++ix) {
        double a = 0.0;
        if (iy >= 1) a += y[(iz * ny1 + iy - 1) * g->n[2] + ix];
        if (iy < ny1) a -= y[(iz * ny1 + iy) * g->n[2] + ix];
        x[IDX(g, iz, iy, ix)] = a / g->h[1];
      }
}
static void dx_fwd(const sipref_grid *g, const double *x, double *y) {
  int64_t nx1 = g->n[2] - 1;
  for (int64_t iz = 0; iz < g->n[0]; ++iz)
    for (int64_t iy = 0; iy < g->n[1]; ++iy)
      for (int64_t ix = 0; ix < nx1; ++ix)
        y[(iz * g->n[1] + iy) * nx1 + ix] =
            (x[IDX(g, iz, iy, ix + 1)] - x[IDX(g, iz, iy, ix)]) / g->h[2];
}
static void dx_adj(const sipref_grid *g, const double *y, double *x) {
  int64_t nx1 = g->n[2] - 1;
  for (int64_t iz = 0; iz < g->n[0]; ++iz)
    for (int64_t iy = 0; iy < g->n[1]; ++iy)
      for (int64_t ix = 0; ix < g->n[2]; ++ix) {
        double a = 0.0;
        if (ix >= 1) a += y[(iz * g->n[1] + iy) * nx1 + ix - 1];
        if (ix < nx1) a -= y[(iz * g->n[1] + iy) * nx1 + ix];
        x[IDX(g, iz, iy, ix)] = a / g->h[2];
      }
}

/* G: 'same' correlation with the kh x kw kernel, zero outside the grid
   (2D grids: the plane is (z, x)); reading L21. */
static void blur_fwd(const sipref_grid *g, const double *K, int kh, int kw,
                     const double *x, double *t) {
  int64_t nz = g->n[0], nx = g->n[2];
  for (int64_t iz = 0; iz < nz; ++iz)
    for (int64_t ix = 0; ix < nx; ++ix) {
      double a = 0.0;
      for (int r = 0; r < kh; ++r)
        for (int c = 0; c < kw; ++c) {
          int64_t jz = iz + r - kh / 2, jx = ix + c - kw / 2;
          if (jz < 0 || jz >= nz || jx < 0 || jx >= nx) continue;
          a += K[r * kw + c] * x[jz * nx + jx];
        }
      t[iz * nx + ix] = a;
    }
}
/* G^T: the same sum with the kernel taps mirrored */
static void blur_adj(const sipref_grid *g, const double *K, int kh, int kw,
                     const double *u, double *x) {
  int64_t nz = g->n[0], nx = g->n[2];
  for (int64_t iz = 0; iz < nz; ++iz)
    for (int64_t ix = 0; ix < nx; ++ix) {
      double a = 0.0;
      for (int r = 0; r < kh; ++r)
        for (int c = 0; c < kw; ++c) {
          int64_t jz = iz - (r - kh / 2), jx = ix - (c - kw / 2);
          if (jz < 0 || jz >= nz || jx < 0 || jx >= nx) continue;
          a += K[r * kw + c] * u[jz * nx + jx];
        }
      x[iz * nx + ix] = a;
    }
}

void sipref_apply_A(const sipref_grid *g, const sipref_set *s, const double *x, double *y) {
  int64_t N = sipref_npts(g);
  switch (s->op) {
    case SIPREF_OP_I: memcpy(y, x, (size_t)N * sizeof(double)); break;
    case SIPREF_OP_DZ: dz_fwd(g, x, y); break;
    case SIPREF_OP_DY: dy_fwd(g, x, y); break;
    case SIPREF_OP_DX: dx_fwd(g, x, y); break;
    case SIPREF_OP_TV: { /* [D_z; D_y; D_x] */
      dz_fwd(g, x, y);
      double *o = y + len_dz(g);
      if (g->ndim == 3) { dy_fwd(g, x, o); o += len_dy(g); }
      dx_fwd(g, x, o);
      break;
    }
    case SIPREF_OP_BLUR_MASK: { /* F x = (G x)[mask] */
      double *t = dalloc(N);
      blur_fwd(g, s->kernel, s->kh, s->kw, x, t);
      int64_t j = 0;
      for (int64_t i = 0; i < N; ++i)
        if (s->mask[i]) y[j++] = t[i];
      free(t);
      break;
    }
  }
}

void sipref_apply_AT(const sipref_grid *g, const sipref_set *s, const double *y, double *x) {
  int64_t N = sipref_npts(g);
  switch (s->op) {
    case SIPREF_OP_I: memcpy(x, y, (size_t)N * sizeof(double)); break;
    case SIPREF_OP_DZ: dz_adj(g, y, x); break;
    case SIPREF_OP_DY: dy_adj(g, y, x); break;
    case SIPREF_OP_DX: dx_adj(g, y, x); break;
    case SIPREF_OP_TV: {
      double *t = dalloc(N);
      dz_adj(g, y, x);
      const double *o = y + len_dz(g);
      if (g->ndim == 3) {
        dy_adj(g, o, t);
        for (int64_t i = 0; i < N; ++i) x[i] += t[i];
        o += len_dy(g);
      }
      dx_adj(g, o, t);
      for (int64_t i = 0; i < N; ++i) x[i] += t[i];
      free(t);
      break;
    }
    case SIPREF_OP_BLUR_MASK: { /* F^T y = G^T (S^T y) */
      double *u = dalloc(N);
      int64_t j = 0;
      for (int64_t i = 0; i < N; ++i) u[i] = s->mask[i] ? y[j++] : 0.0;
      blur_adj(g, s->kernel, s->kh, s->kw, u, x);
      free(u);
      break;
    }
  }
}

/* Eq. 23, applied literally: q = rho_{p+1} p + sum_i rho_i A_i^T (A_i p) */
void sipref_apply_C(const sipref_grid *g, int p, const sipref_set *sets,
                    const double *rho, const double *pv, double *q) {
  int64_t N = sipref_npts(g);
  double *t = dalloc(N);
  for (int64_t j = 0; j < N; ++j) q[j] = rho[p] * pv[j];
  for (int i = 0; i < p; ++i) {
    int64_t M = sipref_op_len(g, &sets[i]);
    double *a = dalloc(M);
    sipref_apply_A(g, &sets[i], pv, a);
    sipref_apply_AT(g, &sets[i], a, t);
    for (int64_t j = 0; j < N; ++j) q[j] += rho[i] * t[j];
    free(a);
  }
  free(t);
}

/* ------------------------------------------------------------------ */
/* projectors, Table 1                                                  */
/* ------------------------------------------------------------------ */
static int cmp_desc(const void *a, const void *b) {
  double x = *(const double *)a, y = *(const double *)b;
  return (x < y) - (x > y);
}

/* l1 ball (Duchi et al. 2008): sort |w| descending into u, find the
   largest j with u_j - (sum_{r<=j} u_r - sigma)/j > 0, theta = (sum_{r<=j}
   u_r - sigma)/j, y = sign(w) max(|w| - theta, 0).  Reading L5. */
static void proj_l1(int64_t M, const double *w, double sigma, double *y) {
  double nrm1 = 0.0;
  for (int64_t i = 0; i < M; ++i) nrm1 += fabs(w[i]);
  if (nrm1 <= sigma) { memcpy(y, w, (size_t)M * sizeof(double)); return; }
  if (sigma <= 0.0) { memset(y, 0, (size_t)M * sizeof(double)); return; }
  double *u = dalloc(M);
  for (int64_t i = 0; i < M; ++i) u[i] = fabs(w[i]);
  qsort(u, (size_t)M, sizeof(double), cmp_desc);
  double cs = 0.0, theta = 0.0;
  for (int64_t j = 0; j < M; ++j) {
    cs += u[j];
    double t = (cs - sigma) / (double)(j + 1);
    if (u[j] - t > 0.0) theta = t;
  }
  for (int64_t i = 0; i < M; ++i) {
    double a = fabs(w[i]) - theta;
    y[i] = a > 0.0 ? (w[i] > 0.0 ? a : -a) : 0.0;
  }
  free(u);
}

/* cardinality (Table 1): keep the k entries of largest |w|; ties go to the
   lowest index (reading L6).  Stable selection by (-|w|, index). */
typedef struct { double a; int64_t i; } keyidx;
static int cmp_keyidx(const void *pa, const void *pb) {
  const keyidx *a = (const keyidx *)pa, *b = (const keyidx *)pb;
  if (a->a > b->a) return -1;
  if (a->a < b->a) return 1;
  return (a->i > b->i) - (a->i < b->i);
}
static void proj_card(int64_t M, const double *w, int64_t k, double *y) {
  if (k >= M) { memcpy(y, w, (size_t)M * sizeof(double)); return; }
  keyidx *t = (keyidx *)malloc((size_t)(M > 0 ? M : 1) * sizeof(keyidx));
  for (int64_t i = 0; i < M; ++i) {
    t[i].a = fabs(w[i]);
    t[i].i = i;
  }
  qsort(t, (size_t)M, sizeof(keyidx), cmp_keyidx);
  memset(y, 0, (size_t)M * sizeof(double));
  for (int64_t j = 0; j < k; ++j) y[t[j].i] = w[t[j].i];
  free(t);
}

/* ------------------------------------------------------------------ */
/* rank and nuclear-norm sets (Table 1): singular values of the */
/* operator's output viewed as a matrix                                   */
/* ------------------------------------------------------------------ */
/* reading L29: 2D grids: the field of A x is one (z, x) matrix; 3D grids:
   one (y, x) matrix per z-plane */
void sipref_matrix_shape(const sipref_grid *g, int op, int64_t *rows, int64_t *cols) {
  int64_t nz = g->n[0], ny = g->n[1], nx = g->n[2];
  int64_t fz = nz - (op == SIPREF_OP_DZ), fy = ny - (op == SIPREF_OP_DY), fx = nx - (op == SIPREF_OP_DX);
  if (g->ndim == 2) { *rows = fz; *cols = fx; }
  else { *rows = fy; *cols = fx; }
}

/* One-sided Jacobi SVD (Hestenes): rotate pairs of columns of X (m x n,
   n <= m, column j at X + j m) until every pair is orthogonal; V (n x n,
   column-major) accumulates the rotations, so X_in V = X_out and the
   singular values are the column norms of X_out. */
static void jacobi_onesided(int64_t m, int64_t n, double *X, double *V) {
  for (int64_t i = 0; i < n * n; ++i) V[i] = 0.0;
  for (int64_t j = 0; j < n; ++j) V[j * n + j] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    int rotated = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = i + 1; j < n; ++j) {
        double *xi = X + i * m, *xj = X + j * m;
        double a = dot(m, xi, xi), b = dot(m, xj, xj), c = dot(m, xi, xj);
        if (c == 0.0 || fabs(c) <= 1e-15 * sqrt(a * b)) continue;
        double zeta = (b - a) / (2.0 * c);
        double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int64_t r = 0; r < m; ++r) {
          double u = xi[r], v = xj[r];
          xi[r] = cs * u - sn * v;
          xj[r] = sn * u + cs * v;
        }
        double *vi = V + i * n, *vj = V + j * n;
        for (int64_t r = 0; r < n; ++r) {
          double u = vi[r], v = vj[r];
          vi[r] = cs * u - sn * v;
          vj[r] = sn * u + cs * v;
        }
        rotated = 1;
      }
    if (!rotated) break;
  }
}

/* the matrix a (rows x cols, row-major) as X (m x n column-major, n <= m):
   X = a^T's columns when cols <= rows (X column j = column j of a), else
   the columns of a^T */
static int load_cols(int64_t rows, int64_t cols, const double *a, double *X, int64_t *m, int64_t *n) {
  int tr = cols > rows;              /* wide: work on a^T */
  *m = tr ? cols : rows;
  *n = tr ? rows : cols;
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) {
      if (!tr) X[j * rows + i] = a[i * cols + j];     /* column j of a */
      else X[i * cols + j] = a[i * cols + j];         /* column i of a^T = row i of a */
    }
  return tr;
}

static int cmp_sv(const void *pa, const void *pb) {
  const keyidx *a = (const keyidx *)pa, *b = (const keyidx *)pb;
  if (a->a > b->a) return -1;
  if (a->a < b->a) return 1;
  return (a->i > b->i) - (a->i < b->i);
}

void sipref_svd_values(int64_t rows, int64_t cols, const double *a, double *sv) {
  int64_t m, n;
  double *X = dalloc(rows * cols), *V = NULL;
  load_cols(rows, cols, a, X, &m, &n);
  V = dalloc(n * n);
  jacobi_onesided(m, n, X, V);
  keyidx *t = (keyidx *)malloc((size_t)n * sizeof(keyidx));
  for (int64_t j = 0; j < n; ++j) { t[j].a = nrm2(m, X + j * m); t[j].i = j; }
  qsort(t, (size_t)n, sizeof(keyidx), cmp_sv);
  for (int64_t j = 0; j < n; ++j) sv[j] = t[j].a;
  free(t); free(X); free(V);
}

/* projection of one matrix: a = sum_j lambda_j u_j v_j^T (SVD);
   RANK r: keep the r largest lambda_j (ties: lowest index; Eckart-Young,
   the nearest matrix of rank <= r); NUCLEAR sigma: lambda projected onto
   {sum lambda <= sigma} (lambda >= 0: the l1 ball of Duchi et al.).
   y = sum_j f_j u_j v_j^T = sum_j (f_j / lambda_j) x_j v_j^T with x_j the
   rotated columns (x_j = lambda_j u_j). */
static void proj_matrix(const sipref_set *s, int64_t rows, int64_t cols, const double *a, double *y) {
  int64_t m, n;
  double *X = dalloc(rows * cols);
  int tr = load_cols(rows, cols, a, X, &m, &n);
  double *V = dalloc(n * n);
  jacobi_onesided(m, n, X, V);
  double *lam = dalloc(n), *f = dalloc(n);
  for (int64_t j = 0; j < n; ++j) lam[j] = nrm2(m, X + j * m);
  if (s->type == SIPREF_RANK) {
    keyidx *t = (keyidx *)malloc((size_t)n * sizeof(keyidx));
    for (int64_t j = 0; j < n; ++j) { t[j].a = lam[j]; t[j].i = j; }
    qsort(t, (size_t)n, sizeof(keyidx), cmp_sv);
    for (int64_t q = 0; q < n; ++q) f[t[q].i] = (q < s->k) ? lam[t[q].i] : 0.0;
    free(t);
  } else {
    proj_l1(n, lam, s->sigma, f);    /* lam >= 0, so the l1 ball is the capped simplex */
  }
  double *B = dalloc(m * n);          /* B = X diag(f / lambda) V^T (column-major m x n) */
  for (int64_t j = 0; j < n; ++j) {
    if (lam[j] == 0.0 || f[j] == 0.0) continue;
    double sc = f[j] / lam[j];
    for (int64_t c = 0; c < n; ++c) {
      double w = sc * V[j * n + c];   /* (V^T)[j][c] = V[c][j] = column j entry c */
      for (int64_t r = 0; r < m; ++r) B[c * m + r] += X[j * m + r] * w;
    }
  }
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j)
      y[i * cols + j] = tr ? B[i * cols + j] : B[j * rows + i];
  free(X); free(V); free(lam); free(f); free(B);
}

/* ------------------------------------------------------------------ */
/* orthogonal-transform sets: V = {x :        */
/* ||D x||_1 <= sigma} with D the orthonormal DCT-II of the grid, kept   */
/* inside the set: P_V(x) = D^T P_l1(D x) (reading L30)     */
/* ------------------------------------------------------------------ */
/* X_k = s_k sum_n x_n cos(pi (2n + 1) k / (2 L)), s_0 = sqrt(1/L),
   s_k = sqrt(2/L); along one axis of length L with stride `st` */
#define SIPREF_PI 3.14159265358979323846
static void dct_axis(int64_t L, int64_t count, int64_t st, int64_t outer_st, int64_t inner, int inverse,
                     double *a) {
  double *t = dalloc(L);
  for (int64_t o = 0; o < count; ++o)
    for (int64_t in = 0; in < inner; ++in) {
      double *p = a + o * outer_st + in;
      for (int64_t k = 0; k < L; ++k) {
        double acc = 0.0;
        for (int64_t n = 0; n < L; ++n) {
          int64_t kk = inverse ? n : k, nn = inverse ? k : n;   /* D^T: swap the roles */
          double s = kk == 0 ? sqrt(1.0 / (double)L) : sqrt(2.0 / (double)L);
          acc += s * cos(SIPREF_PI * (double)(2 * nn + 1) * (double)kk / (2.0 * (double)L)) * p[n * st];
        }
        t[k] = acc;
      }
      for (int64_t k = 0; k < L; ++k) p[k * st] = t[k];
    }
  free(t);
}

void sipref_dct(const sipref_grid *g, int inverse, const double *x, double *y) {
  int64_t nz = g->n[0], ny = g->n[1], nx = g->n[2], N = nz * ny * nx;
  memcpy(y, x, (size_t)N * sizeof(double));
  dct_axis(nx, nz * ny, 1, nx, 1, inverse, y);                 /* x: rows of length nx */
  if (g->ndim == 3) dct_axis(ny, nz, nx, ny * nx, nx, inverse, y);   /* y: per plane, stride nx */
  dct_axis(nz, 1, ny * nx, 0, ny * nx, inverse, y);            /* z: stride plane */
}

/* Orthonormal Haar wavelet transform (the paper's "wavelet" example of an
   orthogonal transform; reading L30), full depth, along one axis
   of length L = 2^J: the pyramid step on the leading n entries
       a_i = (u_{2i} + u_{2i+1}) / sqrt(2),  d_i = (u_{2i} - u_{2i+1}) / sqrt(2)
   stores [a, d] and repeats on a with n/2 until n = 1; the output is
   [a_J, d_J, d_{J-1}, ..., d_1].  The inverse undoes the steps in reverse
   order: u_{2i} = (a_i + d_i) / sqrt(2), u_{2i+1} = (a_i - d_i) / sqrt(2). */
static void haar_axis(int64_t L, int64_t count, int64_t st, int64_t outer_st, int64_t inner, int inverse,
                      double *a) {
  double *u = dalloc(L), *t = dalloc(L);
  const double r2 = sqrt(0.5);
  for (int64_t o = 0; o < count; ++o)
    for (int64_t in = 0; in < inner; ++in) {
      double *p = a + o * outer_st + in;
      for (int64_t k = 0; k < L; ++k) u[k] = p[k * st];
      if (!inverse) {
        for (int64_t n = L; n > 1; n /= 2) {
          for (int64_t i = 0; i < n / 2; ++i) {
            t[i] = (u[2 * i] + u[2 * i + 1]) * r2;
            t[n / 2 + i] = (u[2 * i] - u[2 * i + 1]) * r2;
          }
          for (int64_t i = 0; i < n; ++i) u[i] = t[i];
        }
      } else {
        for (int64_t n = 2; n <= L; n *= 2) {
          for (int64_t i = 0; i < n / 2; ++i) {
            t[2 * i] = (u[i] + u[n / 2 + i]) * r2;
            t[2 * i + 1] = (u[i] - u[n / 2 + i]) * r2;
          }
          for (int64_t i = 0; i < n; ++i) u[i] = t[i];
        }
      }
      for (int64_t k = 0; k < L; ++k) p[k * st] = u[k];
    }
  free(u); free(t);
}

void sipref_haar(const sipref_grid *g, int inverse, const double *x, double *y) {
  int64_t nz = g->n[0], ny = g->n[1], nx = g->n[2], N = nz * ny * nx;
  memcpy(y, x, (size_t)N * sizeof(double));
  haar_axis(nx, nz * ny, 1, nx, 1, inverse, y);
  if (g->ndim == 3) haar_axis(ny, nz, nx, ny * nx, nx, inverse, y);
  haar_axis(nz, 1, ny * nx, 0, ny * nx, inverse, y);
}

/* the set's transform: DCT-II (DCT_L1) or Haar (HAAR_L1) */
static void transform(const sipref_grid *g, int type, int inverse, const double *x, double *y) {
  if (type == SIPREF_HAAR_L1) sipref_haar(g, inverse, x, y);
  else sipref_dct(g, inverse, x, y);
}

static void project_whole(const sipref_set *s, int64_t M, const double *w, double *y);

/* fiber length (reading L28): nx (nx - 1 for D_x) for x-fibers, nz
   (nz - 1 for D_z) for z-fibers -- the forward differences of Eq. 8 */
int64_t sipref_fiber_len(const sipref_grid *g, const sipref_set *s) {
  if (s->app_mode == 1) return s->op == SIPREF_OP_DX ? g->n[2] - 1 : g->n[2];
  if (s->app_mode == 2) return s->op == SIPREF_OP_DZ ? g->n[0] - 1 : g->n[0];
  return 0;
}

/* Table 1 projector of set s on w (length M).  app_mode 1 / 2 (P:418, S:202-
   210, reading L28 of DESIGN.md): the output
   field of the (single-block) operator is split into its x-fibers, which are
   consecutive runs of fib_len entries of the compact layout, or its
   z-fibers, fib_len entries at stride M / fib_len; each fiber is projected
   on its own with the set's parameters (k, sigma per fiber). */
void sipref_project(const sipref_set *s, int64_t M, const double *w, double *y) {
  if (s->app_mode == 0 || s->fib_len <= 0) { project_whole(s, M, w, y); return; }
  const int64_t L = s->fib_len, nf = M / L;
  const int64_t stride = s->app_mode == 1 ? 1 : nf;
  double *a = dalloc(L), *b = dalloc(L);
  for (int64_t f = 0; f < nf; ++f) {
    const int64_t base = s->app_mode == 1 ? f * L : f;
    for (int64_t t = 0; t < L; ++t) a[t] = w[base + t * stride];
    project_whole(s, L, a, b);
    for (int64_t t = 0; t < L; ++t) y[base + t * stride] = b[t];
  }
  free(a);
  free(b);
}

static void project_whole(const sipref_set *s, int64_t M, const double *w, double *y) {
  switch (s->type) {
    case SIPREF_BOUNDS: /* l[i] <= (Am)[i] <= u[i]: clamp */
      for (int64_t i = 0; i < M; ++i) {
        double lo = s->lo_vec ? s->lo_vec[i] : s->lo;
        double hi = s->hi_vec ? s->hi_vec[i] : s->hi;
        double v = w[i];
        y[i] = v < lo ? lo : (v > hi ? hi : v);
      }
      break;
    case SIPREF_L1: proj_l1(M, w, s->sigma, y); break;
    case SIPREF_L2: { /* radial scaling */
      double n = nrm2(M, w);
      double f = (n > s->sigma) ? s->sigma / n : 1.0;
      for (int64_t i = 0; i < M; ++i) y[i] = w[i] * f;
      break;
    }
    case SIPREF_ANNULUS: { /* sigma_l <= ||w|| <= sigma_u; L7 at w = 0 */
      double n = nrm2(M, w);
      if (n == 0.0) {
        memset(y, 0, (size_t)M * sizeof(double));
        if (s->sigma_lo > 0.0 && M > 0) y[0] = s->sigma_lo;
        break;
      }
      double f = 1.0;
      if (n > s->sigma_hi) f = s->sigma_hi / n;
      else if (n < s->sigma_lo) f = s->sigma_lo / n;
      for (int64_t i = 0; i < M; ++i) y[i] = w[i] * f;
      break;
    }
    case SIPREF_CARD: proj_card(M, w, s->k, y); break;
    case SIPREF_DCT_L1:
    case SIPREF_HAAR_L1: {   /* D^T P_l1(D w) */
      sipref_grid gg = s->tgrid;
      double *c1 = dalloc(M), *c2 = dalloc(M);
      transform(&gg, s->type, 0, w, c1);
      proj_l1(M, c1, s->sigma, c2);
      transform(&gg, s->type, 1, c2, y);
      free(c1); free(c2);
      break;
    }
    case SIPREF_RANK:
    case SIPREF_NUCLEAR: {   /* every matrix of the view on its own (L29) */
      int64_t mn = s->mrows * s->mcols;
      for (int64_t o = 0; mn > 0 && o + mn <= M; o += mn) proj_matrix(s, s->mrows, s->mcols, w + o, y + o);
      break;
    }
  }
}

/* Eq. 22: prox of 1/2||z - m||^2 with penalty rho: (m + rho w)/(1 + rho) */
void sipref_prox_dist(int64_t N, const double *m, double rho, const double *w, double *y) {
  for (int64_t i = 0; i < N; ++i) y[i] = (m[i] + rho * w[i]) / (1.0 + rho);
}

static int zero_in_set(const sipref_set *s, int64_t M) {
  if (s->type == SIPREF_BOUNDS) {
    for (int64_t i = 0; i < M; ++i) {
      double lo = s->lo_vec ? s->lo_vec[i] : s->lo;
      double hi = s->hi_vec ? s->hi_vec[i] : s->hi;
      if (lo > 0.0 || hi < 0.0) return 0;
    }
    return 1;
  }
  if (s->type == SIPREF_ANNULUS) return s->sigma_lo <= 0.0;
  return 1;
}

/* Eq. 26: ||s - P(s)|| / ||s||; reading L19 when ||s|| = 0 */
double sipref_feas(const sipref_set *s, int64_t M, const double *sv) {
  double den = nrm2(M, sv);
  if (den == 0.0) return zero_in_set(s, M) ? 0.0 : INFINITY;
  double *pr = dalloc(M);
  sipref_project(s, M, sv, pr);
  double num = 0.0;
  for (int64_t i = 0; i < M; ++i) num += (sv[i] - pr[i]) * (sv[i] - pr[i]);
  free(pr);
  return sqrt(num) / den;
}

/* ------------------------------------------------------------------ */
/* CG on C x = b, warm started, Eq. 25 (reading L18)                    */
/* ------------------------------------------------------------------ */
static int cg_core(const sipref_grid *g, int p, const sipref_set *sets, const double *rho,
                   const double *b, double *x, int n_cg, int eq25, double tol_floor,
                   double *tol_out, int *breakdown) {
  int64_t N = sipref_npts(g);
  double *r = dalloc(N), *pv = dalloc(N), *q = dalloc(N);
  int it = 0;
  *breakdown = 0;
  double bn = nrm2(N, b);
  if (bn == 0.0) { /* zero right-hand side gives x = 0 */
    memset(x, 0, (size_t)N * sizeof(double));
    if (tol_out) *tol_out = 0.0;
    goto done;
  }
  sipref_apply_C(g, p, sets, rho, x, q);
  for (int64_t i = 0; i < N; ++i) r[i] = b[i] - q[i];
  double rr = dot(N, r, r);
  /* Eq. 25: stop when ||r||/||b|| < 0.1 ||C x^k - b|| / ||b|| */
  double tol = 0.1 * sqrt(rr) / bn;
  if (tol < tol_floor) tol = tol_floor;
  if (tol_out) *tol_out = tol;
  memcpy(pv, r, (size_t)N * sizeof(double));
  for (int j = 0; j < n_cg; ++j) {
    if (rr == 0.0) break;
    if (eq25 && sqrt(rr) / bn < tol) break;
    sipref_apply_C(g, p, sets, rho, pv, q);
    double pq = dot(N, pv, q);
    if (!(pq > 0.0)) { *breakdown = 1; break; }
    double alpha = rr / pq;
    for (int64_t i = 0; i < N; ++i) x[i] += alpha * pv[i];
    for (int64_t i = 0; i < N; ++i) r[i] -= alpha * q[i];
    double rr_new = dot(N, r, r);
    double beta = rr_new / rr;
    for (int64_t i = 0; i < N; ++i) pv[i] = r[i] + beta * pv[i];
    rr = rr_new;
    ++it;
  }
done:
  free(r); free(pv); free(q);
  return it;
}

int sipref_cg(const sipref_grid *g, int p, const sipref_set *sets, const double *rho,
              const double *b, double *x, int n_cg, int eq25, double *tol_out,
              int *breakdown) {
  int bd = 0;
  int it = cg_core(g, p, sets, rho, b, x, n_cg, eq25, 10.0 * DBL_EPSILON, tol_out, &bd);
  if (breakdown) *breakdown = bd;
  return it;
}

/* ------------------------------------------------------------------ */
/* Algorithm 2, adapt-rho-gamma                             */
/* ------------------------------------------------------------------ */
/* from the six inner products; reading L17 for zero norms */
static int adapt_from_dots(double hv, double hh, double vhvh, double gv, double gg, double vv,
                           double rho, double eps_corr, double *rho_new, double *gamma_new) {
  int a_ok = 0, b_ok = 0;
  double ahat = 0.0, bhat = 0.0;
  if (hh > 0.0 && vhvh > 0.0) {
    double acorr = hv / (sqrt(hh) * sqrt(vhvh));
    if (acorr > eps_corr) {
      double mg = hv / hh, sd = vhvh / hv;
      ahat = (2.0 * mg > sd) ? mg : sd - 0.5 * mg;
      a_ok = 1;
    }
  }
  if (gg > 0.0 && vv > 0.0) {
    double bcorr = gv / (sqrt(gg) * sqrt(vv));
    if (bcorr > eps_corr) {
      double mg = gv / gg, sd = vv / gv;
      bhat = (2.0 * mg > sd) ? mg : sd - 0.5 * mg;
      b_ok = 1;
    }
  }
  if (a_ok && b_ok) {
    double r = sqrt(ahat * bhat);
    *rho_new = r;
    *gamma_new = 1.0 + 2.0 * r / (ahat + bhat);
    return 0;
  }
  if (a_ok) { *rho_new = ahat; *gamma_new = 1.9; return 1; }
  if (b_ok) { *rho_new = bhat; *gamma_new = 1.1; return 2; }
  *rho_new = rho; *gamma_new = 1.5;
  return 3;
}

int sipref_adapt_rho_gamma(int64_t M, const double *v_hat, const double *v_hat0,
                           const double *v, const double *v0,
                           const double *s, const double *s0,
                           const double *y, const double *y0,
                           double rho, double eps_corr, double *rho_new,
                           double *gamma_new) {
  double hv = 0, hh = 0, vhvh = 0, gv = 0, gg = 0, vv = 0;
  for (int64_t i = 0; i < M; ++i) {
    double dvh = v_hat[i] - v_hat0[i];  /* Delta v-hat */
    double dv = v[i] - v0[i];           /* Delta v     */
    double dh = s[i] - s0[i];           /* Delta h-hat */
    double dg = -(y[i] - y0[i]);        /* Delta g-hat */
    hv += dh * dvh; hh += dh * dh; vhvh += dvh * dvh;
    gv += dg * dv; gg += dg * dg; vv += dv * dv;
  }
  return adapt_from_dots(hv, hh, vhvh, gv, gg, vv, rho, eps_corr, rho_new, gamma_new);
}

/* ------------------------------------------------------------------ */
/* set resolution: relative parameters (readings L4, L23)               */
/* ------------------------------------------------------------------ */
void sipref_resolve_set(const sipref_grid *g, const sipref_set *in, const double *m,
                        sipref_set *out) {
  *out = *in;
  out->fib_len = sipref_fiber_len(g, in);
  sipref_matrix_shape(g, in->op, &out->mrows, &out->mcols);
  out->tgrid = *g;
  if (!in->relative) return;
  int64_t M = sipref_op_len(g, in);
  double *a = dalloc(M);
  sipref_apply_A(g, in, m, a);
  double n1 = 0.0;
  for (int64_t i = 0; i < M; ++i) n1 += fabs(a[i]);
  double n2 = nrm2(M, a);
  free(a);
  if (in->type == SIPREF_L1) out->sigma = in->sigma * n1;
  if (in->type == SIPREF_L2) out->sigma = in->sigma * n2;
  if (in->type == SIPREF_ANNULUS) {
    out->sigma_lo = in->sigma_lo * n2;
    out->sigma_hi = in->sigma_hi * n2;
  }
  if (in->type == SIPREF_DCT_L1 || in->type == SIPREF_HAAR_L1) {   /* sigma = frac x ||D m||_1 (reading L30) */
    double *am = dalloc(M), *cm = dalloc(M), n1d = 0.0;
    sipref_apply_A(g, in, m, am);
    transform(g, in->type, 0, am, cm);
    for (int64_t j = 0; j < M; ++j) n1d += fabs(cm[j]);
    out->sigma = in->sigma * n1d;
    free(am); free(cm);
  }
  if (in->type == SIPREF_NUCLEAR) {   /* sigma = frac x sum of the nuclear norms of A m's matrices */
    int64_t r, cc;
    sipref_matrix_shape(g, in->op, &r, &cc);
    int64_t mn = r * cc, q = r < cc ? r : cc;
    double *sv = dalloc(q), nuc = 0.0;
    double *am = dalloc(M);
    sipref_apply_A(g, in, m, am);
    for (int64_t o = 0; o + mn <= M; o += mn) {
      sipref_svd_values(r, cc, am + o, sv);
      for (int64_t j = 0; j < q; ++j) nuc += sv[j];
    }
    out->sigma = in->sigma * nuc;
    free(sv); free(am);
  }
  if (in->type == SIPREF_CARD)   /* per fiber: a fraction of the fiber length */
    out->k = (int64_t)floor(in->k_frac * (double)(in->app_mode ? out->fib_len : M));
  out->relative = 0;
}

/* ------------------------------------------------------------------ */
/* support fingerprint of a cardinality set (test instrument, not part of */
/* the method): entry j of A x (compact layout) belongs to block b at     */
/* grid point (iz, iy, ix); its key is splitmix64(b N + grid index).       */
/* ------------------------------------------------------------------ */
static uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static int64_t owner_point(const sipref_grid *g, int blk_op, int64_t j) {
  int64_t ny = g->n[1], nx = g->n[2];
  switch (blk_op) {
    case SIPREF_OP_DY: { int64_t iz = j / ((ny - 1) * nx), r = j % ((ny - 1) * nx);
                         return (iz * ny + r / nx) * nx + r % nx; }
    case SIPREF_OP_DX: return (j / (nx - 1)) * nx + j % (nx - 1);
    default: return j;  /* I and D_z: compact index = grid index */
  }
}
uint64_t sipref_supp_key(const sipref_grid *g, int op, int64_t j) {
  int64_t N = sipref_npts(g);
  if (op == SIPREF_OP_TV) {
    int b = 0;
    if (j >= len_dz(g)) {
      j -= len_dz(g); b = 1;
      if (g->ndim == 3) {
        if (j < len_dy(g)) return splitmix64((uint64_t)(N + owner_point(g, SIPREF_OP_DY, j)));
        j -= len_dy(g); b = 2;
      }
      return splitmix64((uint64_t)(b * N + owner_point(g, SIPREF_OP_DX, j)));
    }
    return splitmix64((uint64_t)j);
  }
  return splitmix64((uint64_t)owner_point(g, op, j));
}

/* ------------------------------------------------------------------ */
/* Algorithm 1, PARSDMM                                                 */
/* ------------------------------------------------------------------ */
static int parsdmm_run(const sipref_grid *g, int p, const sipref_set *in_sets,
                       const sipref_options *o, double tol_floor, const double *m, double *x,
                       const double *init_x, double *const *init_y, double *const *init_v,
                       const double *init_rho, const double *init_gamma,
                       double *const *out_y, double *const *out_v, sipref_log *log) {
  int64_t N = sipref_npts(g);
  int P = p + 1; /* p sets plus the distance block A_{p+1} = I (Eq. 17) */
  sipref_set *sets = (sipref_set *)calloc((size_t)P, sizeof(sipref_set));
  int64_t *M = (int64_t *)calloc((size_t)P, sizeof(int64_t));
  for (int i = 0; i < p; ++i) {
    sipref_resolve_set(g, &in_sets[i], m, &sets[i]);
    M[i] = sipref_op_len(g, &sets[i]);
  }
  sets[p].op = SIPREF_OP_I;
  M[p] = N;

  double **y = (double **)calloc((size_t)P, sizeof(double *));
  double **v = (double **)calloc((size_t)P, sizeof(double *));
  double **s = (double **)calloc((size_t)P, sizeof(double *));
  double **vh = (double **)calloc((size_t)P, sizeof(double *));
  double **vh0 = (double **)calloc((size_t)P, sizeof(double *));
  double **v0 = (double **)calloc((size_t)P, sizeof(double *));
  double **s0 = (double **)calloc((size_t)P, sizeof(double *));
  double **y0 = (double **)calloc((size_t)P, sizeof(double *));
  double *rho = dalloc(P), *gam = dalloc(P);
  double *xbar = NULL, *w = NULL, *yn = NULL;
  int64_t Mmax = N;
  for (int i = 0; i < P; ++i) if (M[i] > Mmax) Mmax = M[i];
  xbar = dalloc(Mmax); w = dalloc(Mmax); yn = dalloc(Mmax);

  /* initialisation, reading L13 */
  if (init_x) memcpy(x, init_x, (size_t)N * sizeof(double));
  else memcpy(x, m, (size_t)N * sizeof(double));
  for (int i = 0; i < P; ++i) {
    y[i] = dalloc(M[i]); v[i] = dalloc(M[i]); s[i] = dalloc(M[i]);
    vh[i] = dalloc(M[i]); vh0[i] = dalloc(M[i]); v0[i] = dalloc(M[i]);
    s0[i] = dalloc(M[i]); y0[i] = dalloc(M[i]);
    if (init_y) memcpy(y[i], init_y[i], (size_t)M[i] * sizeof(double));
    else if (i < p) sipref_apply_A(g, &sets[i], m, y[i]);
    else memcpy(y[i], m, (size_t)N * sizeof(double));
    if (init_v) memcpy(v[i], init_v[i], (size_t)M[i] * sizeof(double));
    rho[i] = init_rho ? init_rho[i] : o->rho0;
    gam[i] = init_gamma ? init_gamma[i] : o->gamma0;
  }
  /* history of x for Eq. 27: starts as [x^1] */
  int S = o->hist_s;
  double **hist = (double **)calloc((size_t)S, sizeof(double *));
  for (int j = 0; j < S; ++j) hist[j] = dalloc(N);
  int hist_count = 1, hist_head = 0; /* hist[head] = newest */
  memcpy(hist[0], x, (size_t)N * sizeof(double));

  double *b = dalloc(N), *t = dalloc(N), *u = dalloc(Mmax);
  int first_adapt = 1, converged = 0, k = 0, cg_total = 0, breakdown = 0;
  double r_evol = INFINITY;
  double *r_feas = dalloc(p > 0 ? p : 1);
  for (int i = 0; i < p; ++i) r_feas[i] = INFINITY;

  for (k = 1; k <= o->max_iter; ++k) {
    /* x^{k+1} = C^{-1} sum_i A_i^T (rho_i y_i + v_i), Eq. 21 line 1 */
    memset(b, 0, (size_t)N * sizeof(double));
    for (int i = 0; i < P; ++i) {
      for (int64_t j = 0; j < M[i]; ++j) u[j] = rho[i] * y[i][j] + v[i][j];
      if (i < p) sipref_apply_AT(g, &sets[i], u, t);
      else memcpy(t, u, (size_t)N * sizeof(double));
      for (int64_t j = 0; j < N; ++j) b[j] += t[j];
    }
    int bd = 0;
    int it = cg_core(g, p, sets, rho, b, x, o->n_cg, o->eq25, tol_floor, NULL, &bd);
    breakdown |= bd;
    cg_total += it;
    if (log && log->cg_per_iter) log->cg_per_iter[k - 1] = it;

    int adapt = (o->adapt_every <= 1) || (k % o->adapt_every == 1);
    /* FOR i = 1..p+1 (Alg. 1) */
    for (int i = 0; i < P; ++i) {
      if (i < p) sipref_apply_A(g, &sets[i], x, s[i]);           /* s = A x */
      else memcpy(s[i], x, (size_t)N * sizeof(double));
      for (int64_t j = 0; j < M[i]; ++j) {
        xbar[j] = gam[i] * s[i][j] + (1.0 - gam[i]) * y[i][j];  /* relaxation */
        w[j] = xbar[j] - v[i][j] / rho[i];
      }
      if (i < p) sipref_project(&sets[i], M[i], w, yn);        /* y = P_C(w) */
      else sipref_prox_dist(N, m, rho[i], w, yn);               /* Eq. 22 */
      if (adapt) /* Alg. 2 line 1 with the OLD y and v (reading L10) */
        for (int64_t j = 0; j < M[i]; ++j) vh[i][j] = v[i][j] + rho[i] * (y[i][j] - s[i][j]);
      /* dual update, Eq. 21 line 4: v + rho (y - x-bar) = rho (y - w) since
         w = x-bar - v/rho.  The second form is exact (v = 0) when the
         constraint is inactive (y = w); the first leaves rounding noise that
         Algorithm 2 would correlate (reading L26). */
      for (int64_t j = 0; j < M[i]; ++j) {
        v[i][j] = rho[i] * (yn[j] - w[j]);
        y[i][j] = yn[j];
      }
    }

    if (log && log->supp_hash)
      for (int i = 0; i < p; ++i) {
        uint64_t hsum = 0;
        if (sets[i].type == SIPREF_CARD)
          for (int64_t j = 0; j < M[i]; ++j)
            if (y[i][j] != 0.0) hsum += sipref_supp_key(g, sets[i].op, j);
        log->supp_hash[(size_t)(k - 1) * p + i] = hsum;
      }

    /* stopping conditions, Eqs. 26-28, every check_every iterations */
    if (o->check_every > 0 && k % o->check_every == 0) {
      int feas_ok = 1;
      for (int i = 0; i < p; ++i) {
        r_feas[i] = sipref_feas(&sets[i], M[i], s[i]);
        if (!(r_feas[i] < o->eps_feas)) feas_ok = 0;
      }
      double xn = nrm2(N, x), mx = 0.0;
      for (int j = 0; j < hist_count; ++j) {
        const double *hj = hist[(hist_head - j + S) % S];
        double d = 0.0;
        for (int64_t q = 0; q < N; ++q) d += (x[q] - hj[q]) * (x[q] - hj[q]);
        d = sqrt(d);
        if (d > mx) mx = d;
      }
      r_evol = (xn > 0.0) ? mx / xn : (mx > 0.0 ? INFINITY : 0.0);
      if (log && log->r_evol_trace) log->r_evol_trace[k - 1] = r_evol;
      if (log && log->r_feas_trace)
        for (int i = 0; i < p; ++i) log->r_feas_trace[(size_t)(k - 1) * p + i] = r_feas[i];
      if (r_evol < o->eps_evol && feas_ok) {
        converged = 1;
        if (!o->fixed_work) {
          if (log && log->branch)
            for (int i = 0; i < P; ++i) log->branch[(size_t)(k - 1) * P + i] = -1;
          if (log && log->rho_trace)
            for (int i = 0; i < P; ++i) {
              log->rho_trace[(size_t)(k - 1) * P + i] = rho[i];
              log->gamma_trace[(size_t)(k - 1) * P + i] = gam[i];
            }
          break;
        }
      }
    } else {
      if (log && log->r_evol_trace) log->r_evol_trace[k - 1] = NAN;
      if (log && log->r_feas_trace)
        for (int i = 0; i < p; ++i) log->r_feas_trace[(size_t)(k - 1) * p + i] = NAN;
    }
    /* push x^{k+1} into the history */
    hist_head = (hist_head + 1) % S;
    memcpy(hist[hist_head], x, (size_t)N * sizeof(double));
    if (hist_count < S) ++hist_count;

    /* adapt rho, gamma when mod(k, 2) = 1 */
    if (log && log->branch)
      for (int i = 0; i < P; ++i) log->branch[(size_t)(k - 1) * P + i] = -1;
    if (adapt) {
      if (!first_adapt) {
        for (int i = 0; i < P; ++i) {
          double rn, gn;
          int br = sipref_adapt_rho_gamma(M[i], vh[i], vh0[i], v[i], v0[i], s[i], s0[i],
                                          y[i], y0[i], rho[i], o->eps_corr, &rn, &gn);
          if (gn < 1.0) gn = 1.0;              /* reading L15 */
          if (gn > o->gamma_max) gn = o->gamma_max;
          rho[i] = rn; gam[i] = gn;
          if (log && log->branch) log->branch[(size_t)(k - 1) * P + i] = br;
        }
        /* reading L16: keep rho_i / rho_{p+1} within [1/cap, cap] */
        for (int i = 0; i < p; ++i) {
          double lo = rho[p] / o->rho_ratio_cap, hi = rho[p] * o->rho_ratio_cap;
          if (rho[i] < lo) rho[i] = lo;
          if (rho[i] > hi) rho[i] = hi;
        }
      }
      first_adapt = 0;
      /* snapshot (v-hat, v, s, y)^{k0} for the next call */
      for (int i = 0; i < P; ++i) {
        memcpy(vh0[i], vh[i], (size_t)M[i] * sizeof(double));
        memcpy(v0[i], v[i], (size_t)M[i] * sizeof(double));
        memcpy(s0[i], s[i], (size_t)M[i] * sizeof(double));
        memcpy(y0[i], y[i], (size_t)M[i] * sizeof(double));
      }
    }
    if (log && log->rho_trace)
      for (int i = 0; i < P; ++i) {
        log->rho_trace[(size_t)(k - 1) * P + i] = rho[i];
        log->gamma_trace[(size_t)(k - 1) * P + i] = gam[i];
      }
  }
  int iters = (k > o->max_iter) ? o->max_iter : k;

  if (log) {
    log->iterations = iters;
    log->cg_total = cg_total;
    log->converged = converged;
    log->breakdown = breakdown;
    log->r_evol = r_evol;
    if (log->r_feas) for (int i = 0; i < p; ++i) log->r_feas[i] = r_feas[i];
    if (log->rho) for (int i = 0; i < P; ++i) log->rho[i] = rho[i];
    if (log->gamma) for (int i = 0; i < P; ++i) log->gamma[i] = gam[i];
  }
  for (int i = 0; i < P; ++i) {
    if (out_y) memcpy(out_y[i], y[i], (size_t)M[i] * sizeof(double));
    if (out_v) memcpy(out_v[i], v[i], (size_t)M[i] * sizeof(double));
    free(y[i]); free(v[i]); free(s[i]); free(vh[i]); free(vh0[i]); free(v0[i]);
    free(s0[i]); free(y0[i]);
  }
  for (int j = 0; j < S; ++j) free(hist[j]);
  free(hist); free(y); free(v); free(s); free(vh); free(vh0); free(v0); free(s0); free(y0);
  free(rho); free(gam); free(xbar); free(w); free(yn); free(b); free(t); free(u);
  free(r_feas); free(sets); free(M);
  return converged ? 0 : 1;
}

int sipref_parsdmm(const sipref_grid *g, int p, const sipref_set *sets,
                   const sipref_options *o, const double *m, double *x,
                   const double *init_x, double *const *init_y, double *const *init_v,
                   const double *init_rho, const double *init_gamma,
                   double *const *out_y, double *const *out_v, sipref_log *log) {
  return parsdmm_run(g, p, sets, o, o->cg_tol_floor, m, x, init_x, init_y, init_v,
                     init_rho, init_gamma, out_y, out_v, log);
}

/* ------------------------------------------------------------------ */
/* Algorithm 3, multilevel PARSDMM                                      */
/* ------------------------------------------------------------------ */
static sipref_grid coarsen_grid(const sipref_grid *f) {
  sipref_grid c = *f;
  c.n[0] = f->n[0] / 2; c.h[0] = f->h[0] * 2.0;
  if (f->ndim == 3) { c.n[1] = f->n[1] / 2; c.h[1] = f->h[1] * 2.0; }
  c.n[2] = f->n[2] / 2; c.h[2] = f->h[2] * 2.0;
  return c;
}

/* "anti-alias filtering and subsampling": mean of each 2x2(x2)
   block, then stride 2 (reading L23) */
void sipref_restrict(const sipref_grid *fine, const double *f, double *c) {
  sipref_grid cg = coarsen_grid(fine);
  int by = (fine->ndim == 3) ? 2 : 1;
  double inv = 1.0 / (double)(2 * by * 2);
  for (int64_t iz = 0; iz < cg.n[0]; ++iz)
    for (int64_t iy = 0; iy < cg.n[1]; ++iy)
      for (int64_t ix = 0; ix < cg.n[2]; ++ix) {
        double a = 0.0;
        for (int dz = 0; dz < 2; ++dz)
          for (int dy = 0; dy < by; ++dy)
            for (int dx = 0; dx < 2; ++dx)
              a += f[IDX(fine, 2 * iz + dz, by * iy + dy, 2 * ix + dx)];
        c[IDX(&cg, iz, iy, ix)] = a * inv;
      }
}

/* (tri)linear interpolation of an image of shape (cz,cy,cx) onto
   (fz,fy,fx), align-corners (reading L23; "interpolate as images") */
static void axis_w(int64_t i, int64_t nf, int64_t nc, int64_t *i0, int64_t *i1, double *t) {
  double pos = (nf > 1 && nc > 1) ? (double)i * (double)(nc - 1) / (double)(nf - 1) : 0.0;
  int64_t a = (int64_t)floor(pos);
  if (a > nc - 1) a = nc - 1;
  *i0 = a;
  *i1 = (a + 1 < nc) ? a + 1 : a;
  *t = pos - (double)a;
}
void sipref_interp(int64_t cz, int64_t cy, int64_t cx, const double *c,
                   int64_t fz, int64_t fy, int64_t fx, double *f) {
  for (int64_t iz = 0; iz < fz; ++iz) {
    int64_t z0, z1; double tz;
    axis_w(iz, fz, cz, &z0, &z1, &tz);
    for (int64_t iy = 0; iy < fy; ++iy) {
      int64_t y0, y1; double ty;
      axis_w(iy, fy, cy, &y0, &y1, &ty);
      for (int64_t ix = 0; ix < fx; ++ix) {
        int64_t x0, x1; double tx;
        axis_w(ix, fx, cx, &x0, &x1, &tx);
#define C_(a, b, d) c[((a) * cy + (b)) * cx + (d)]
        double v00 = C_(z0, y0, x0) * (1.0 - tx) + C_(z0, y0, x1) * tx;
        double v01 = C_(z0, y1, x0) * (1.0 - tx) + C_(z0, y1, x1) * tx;
        double v10 = C_(z1, y0, x0) * (1.0 - tx) + C_(z1, y0, x1) * tx;
        double v11 = C_(z1, y1, x0) * (1.0 - tx) + C_(z1, y1, x1) * tx;
#undef C_
        double v0 = v00 * (1.0 - ty) + v01 * ty;
        double v1 = v10 * (1.0 - ty) + v11 * ty;
        f[(iz * fy + iy) * fx + ix] = v0 * (1.0 - tz) + v1 * tz;
      }
    }
  }
}

/* interpolate the field of one operator (block by block for TV): each block
   is an image of its own shape ("as images"; reading L23), e.g.
   D_z's (nz-1) x ny x nx */
void sipref_prolong_field(const sipref_grid *cgd, const sipref_grid *fgd, int op,
                          const double *c, double *f) {
  int64_t cz = cgd->n[0], cy = cgd->n[1], cx = cgd->n[2];
  int64_t fz = fgd->n[0], fy = fgd->n[1], fx = fgd->n[2];
  switch (op) {
    case SIPREF_OP_I: sipref_interp(cz, cy, cx, c, fz, fy, fx, f); break;
    case SIPREF_OP_DZ: sipref_interp(cz - 1, cy, cx, c, fz - 1, fy, fx, f); break;
    case SIPREF_OP_DY: sipref_interp(cz, cy - 1, cx, c, fz, fy - 1, fx, f); break;
    case SIPREF_OP_DX: sipref_interp(cz, cy, cx - 1, c, fz, fy, fx - 1, f); break;
    case SIPREF_OP_TV: {
      sipref_interp(cz - 1, cy, cx, c, fz - 1, fy, fx, f);
      c += (cz - 1) * cy * cx; f += (fz - 1) * fy * fx;
      if (cgd->ndim == 3) {
        sipref_interp(cz, cy - 1, cx, c, fz, fy - 1, fx, f);
        c += cz * (cy - 1) * cx; f += fz * (fy - 1) * fx;
      }
      sipref_interp(cz, cy, cx - 1, c, fz, fy, fx - 1, f);
      break;
    }
  }
}

int sipref_parsdmm_multilevel(const sipref_grid *g, int p, const sipref_set *sets,
                              const sipref_options *o, int n_levels,
                              const double *m, double *x, sipref_log *logs) {
  if (n_levels < 1) return -1;
  for (int i = 0; i < p; ++i)
    if (sets[i].op == SIPREF_OP_BLUR_MASK || sets[i].lo_vec || sets[i].hi_vec) return -2;
  int P = p + 1;
  sipref_grid *gr = (sipref_grid *)calloc((size_t)n_levels, sizeof(sipref_grid));
  double **ml = (double **)calloc((size_t)n_levels, sizeof(double *));
  gr[0] = *g;
  ml[0] = (double *)m;
  for (int l = 1; l < n_levels; ++l) {
    gr[l] = coarsen_grid(&gr[l - 1]);
    ml[l] = dalloc(sipref_npts(&gr[l]));
    sipref_restrict(&gr[l - 1], ml[l - 1], ml[l]);
  }
  double *xc = NULL, **yc = NULL, **vc = NULL;
  double *rho = dalloc(P), *gam = dalloc(P);
  int status = 0;
  for (int l = n_levels - 1; l >= 0; --l) {
    const sipref_grid *gl = &gr[l];
    int64_t Nl = sipref_npts(gl);
    double *xl = (l == 0) ? x : dalloc(Nl);
    double **yl = (double **)calloc((size_t)P, sizeof(double *));
    double **vl = (double **)calloc((size_t)P, sizeof(double *));
    int64_t *Ml = (int64_t *)calloc((size_t)P, sizeof(int64_t));
    for (int i = 0; i < P; ++i) {
      Ml[i] = (i < p) ? sipref_op_len(gl, &sets[i]) : Nl;
      yl[i] = dalloc(Ml[i]);
      vl[i] = dalloc(Ml[i]);
    }
    double *init_x = dalloc(Nl);
    if (l == n_levels - 1) {
      /* coarsest: x = m_L, y_i = v_i = 0 (reading L13) */
      memcpy(init_x, ml[l], (size_t)Nl * sizeof(double));
      for (int i = 0; i < P; ++i) { rho[i] = o->rho0; gam[i] = o->gamma0; }
    } else {
      const sipref_grid *gc = &gr[l + 1];
      sipref_prolong_field(gc, gl, SIPREF_OP_I, xc, init_x);
      for (int i = 0; i < P; ++i) {
        int op = (i < p) ? sets[i].op : SIPREF_OP_I;
        sipref_prolong_field(gc, gl, op, yc[i], yl[i]);
        sipref_prolong_field(gc, gl, op, vc[i], vl[i]);
      }
    }
    sipref_log *lg = logs ? &logs[l] : NULL;
    double *lrho = NULL, *lgam = NULL;
    sipref_log tmp;
    if (!lg) { memset(&tmp, 0, sizeof(tmp)); lg = &tmp; }
    lrho = lg->rho; lgam = lg->gamma;
    double *rbuf = dalloc(P), *gbuf = dalloc(P);
    lg->rho = rbuf; lg->gamma = gbuf;
    int st = sipref_parsdmm(gl, p, sets, o, ml[l], xl, init_x, yl, vl, rho, gam, yl, vl, lg);
    /* rho and gamma carry over to the next level (reading L23) */
    memcpy(rho, rbuf, (size_t)P * sizeof(double));
    memcpy(gam, gbuf, (size_t)P * sizeof(double));
    if (lrho) memcpy(lrho, rbuf, (size_t)P * sizeof(double));
    if (lgam) memcpy(lgam, gbuf, (size_t)P * sizeof(double));
    lg->rho = lrho; lg->gamma = lgam;
    free(rbuf); free(gbuf);
    if (l == 0) status = st;
    free(init_x);
    if (xc) free(xc);
    if (yc) { for (int i = 0; i < P; ++i) { free(yc[i]); free(vc[i]); } free(yc); free(vc); }
    xc = (l == 0) ? NULL : xl;
    yc = yl; vc = vl;
    free(Ml);
  }
  if (yc) { for (int i = 0; i < P; ++i) { free(yc[i]); free(vc[i]); } free(yc); free(vc); }
  for (int l = 1; l < n_levels; ++l) free(ml[l]);
  free(ml); free(gr); free(rho); free(gam);
  return status;
}

/* ------------------------------------------------------------------ */
/* Algorithm 4, parallel Dykstra, Fig. 1 comparator         */
/* ------------------------------------------------------------------ */
int sipref_dykstra(const sipref_grid *g, int p, const sipref_set *in_sets, const sipref_options *inner,
                   int max_outer, double tol, const double *m, double *x, sipref_dykstra_log *log) {
  int64_t N = sipref_npts(g);
  sipref_set *sets = (sipref_set *)calloc((size_t)(p > 0 ? p : 1), sizeof(sipref_set));
  for (int i = 0; i < p; ++i) sipref_resolve_set(g, &in_sets[i], m, &sets[i]);   /* from m, once */
  double **v = (double **)calloc((size_t)p, sizeof(double *));
  double **y = (double **)calloc((size_t)p, sizeof(double *));
  double *xo = dalloc(N);
  memcpy(x, m, (size_t)N * sizeof(double));                          /* 0a */
  for (int i = 0; i < p; ++i) {                                      /* 0b */
    v[i] = dalloc(N); y[i] = dalloc(N);
    memcpy(v[i], x, (size_t)N * sizeof(double));
  }
  const double w = 1.0 / (double)p;                                  /* 0c */
  int k;
  for (k = 1; k <= max_outer; ++k) {
    int cg_max = 0, l1p = 0;
    for (int i = 0; i < p; ++i) {                                    /* 1 */
      int it = 0, cg = 0;
      if (sets[i].op == SIPREF_OP_I) {
        sipref_project(&sets[i], N, v[i], y[i]);
        it = 1;
      } else {
        sipref_log lg;
        memset(&lg, 0, sizeof(lg));
        sipref_parsdmm(g, 1, &sets[i], inner, v[i], y[i], NULL, NULL, NULL, NULL, NULL, NULL, NULL, &lg);
        it = lg.iterations;
        cg = lg.cg_total;
      }
      if (cg > cg_max) cg_max = cg;
      if (sets[i].type == SIPREF_L1) l1p += it;
      if (log && log->inner_iters) log->inner_iters[(size_t)(k - 1) * p + i] = it;
    }
    memcpy(xo, x, (size_t)N * sizeof(double));
    for (int64_t j = 0; j < N; ++j) {                                /* 2 */
      double a = 0.0;
      for (int i = 0; i < p; ++i) a += w * y[i][j];
      x[j] = a;
    }
    for (int i = 0; i < p; ++i)                                      /* 3 */
      for (int64_t j = 0; j < N; ++j) v[i][j] = x[j] + v[i][j] - y[i][j];
    double d = 0.0;
    for (int64_t j = 0; j < N; ++j) d += (x[j] - xo[j]) * (x[j] - xo[j]);
    double xn = nrm2(N, x);
    double re = xn > 0.0 ? sqrt(d) / xn : 0.0;
    if (log) {
      if (log->cg_max) log->cg_max[k - 1] = cg_max;
      if (log->l1_proj) log->l1_proj[k - 1] = l1p;
      if (log->r_evol) log->r_evol[k - 1] = re;
      if (log->r_feas)
        for (int i = 0; i < p; ++i) {
          int64_t M = sipref_op_len(g, &sets[i]);
          double *a = dalloc(M);
          sipref_apply_A(g, &sets[i], x, a);
          log->r_feas[(size_t)(k - 1) * p + i] = sipref_feas(&sets[i], M, a);
          free(a);
        }
    }
    if (re < tol) break;
  }
  if (log) log->iterations = k > max_outer ? max_outer : k;
  for (int i = 0; i < p; ++i) { free(v[i]); free(y[i]); }
  free(v); free(y); free(xo); free(sets);
  return k > max_outer ? 1 : 0;
}
