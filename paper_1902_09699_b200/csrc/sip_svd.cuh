// sip_svd.cuh -- rank and nuclear-norm sets (Table 1; SURVEY
// 8(f) NEXT-2) on the device: the projection of every matrix of the view of
// A x (reading L29: 2D grids one (z, x) matrix; 3D grids one (y, x) matrix
// per z-plane) by a batched one-sided Jacobi SVD, one CTA per matrix.
//
//   load      X (m x n, column-major, n = min(rows, cols); a wide matrix is
//             taken transposed) in fp64 scratch, V = I (n x n)
//   sweeps    round-robin (circle) ordering: each round pairs all columns
//             disjointly, one warp per pair at a time: the three inner
//             products, the Jacobi rotation that makes the pair orthogonal,
//             applied to both columns of X and of V; until a sweep rotates
//             nothing (|x_i . x_j| <= 1e-15 |x_i| |x_j| for every pair)
//   values    lambda_j = |x_j| (X V = U diag(lambda), the rotated columns)
//   project   rank r: f_j = lambda_j for the r largest (ties: lowest index),
//             else 0 (Eckart-Young); nuclear sigma: f = the l1-ball
//             projection of lambda (lambda >= 0: max(lambda - theta, 0),
//             Duchi's active set)
//   write     P(A) = X diag(f / lambda) V^T, then (which = 0) y = P(w),
//             v = rho (y - w) and Alg. 2's beta-side products; (which = 1,
//             check iterations) the Eq. 26 numerator |s - P(s)|^2; (which =
//             2, initialisation) the nuclear norm of A m for a relative radius
//
// fp64 inside (the rotations need it); the fields stay in the grid dtype.
#pragma once
#include "sip_pass.cuh"

namespace sip {

constexpr int SVD_BLOCK = 512;
constexpr int SVD_NMAX = 2048;     // min(rows, cols) limit (shared lambda / f)

struct MatView {
  int rows, cols, nmat;            // matrix shape and count
  int m, n, tr;                    // X = a (tr = 0) or a^T (tr = 1): m x n, n <= m
};

__host__ __device__ inline MatView mat_view(int ndim, int nz, int ny, int nx, int prim) {
  const int fz = nz - (prim == PRIM_Z), fy = ny - (prim == PRIM_Y), fx = nx - (prim == PRIM_X);
  MatView v;
  if (ndim == 2) { v.rows = fz; v.cols = fx; v.nmat = 1; }
  else { v.rows = fy; v.cols = fx; v.nmat = fz; }
  v.tr = v.cols > v.rows;
  v.m = v.tr ? v.cols : v.rows;
  v.n = v.tr ? v.rows : v.cols;
  return v;
}

// grid point of matrix element (r, c) of matrix b (padded field layout)
__device__ __forceinline__ int64_t mat_pt(const Geo& g, int b, int r, int c) {
  return g.ndim == 2 ? (int64_t)r * g.nx + c : (int64_t)b * g.plane + (int64_t)r * g.nx + c;
}

// every lane gets the warp total (the rotation is computed by all lanes)
__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- thread-block cluster helpers (one matrix per cluster of CL CTAs) ----
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// all threads of every CTA of the cluster; release / acquire at cluster scope
__device__ __forceinline__ void cl_sync(int cl) {
  if (cl == 1) { __syncthreads(); return; }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// address of `p` (this CTA's shared memory) in CTA `r` of the cluster
__device__ __forceinline__ unsigned cl_map(const void* p, unsigned r) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(r));
  return ra;
}
__device__ __forceinline__ void cl_st(unsigned ra, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}
__device__ __forceinline__ int cl_ld(unsigned ra) {
  int v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
  return v;
}

// One Jacobi step on the column pair (xi, xj) of length m (and the same
// rotation on V's columns vi, vj of length n), by one warp.  Lane l holds
// rows l, l + 32, ... (accumulated in that order, as a plain lane loop
// would); columns of at most 32 R rows stay in registers between the inner
// products and the rotation (one L2 round trip per column).  Returns whether
// the pair was rotated.
template <int R>
__device__ __forceinline__ void rot_cols(double* a, double* b, int len, int lane, double cs, double sn) {
  for (int r0 = 0; r0 < len; r0 += 32 * R) {
    double u[R], v[R];
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int r = r0 + lane + 32 * e;
      u[e] = r < len ? __ldcg(a + r) : 0.0;
      v[e] = r < len ? __ldcg(b + r) : 0.0;
    }
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int r = r0 + lane + 32 * e;
      if (r < len) { a[r] = cs * u[e] - sn * v[e]; b[r] = sn * u[e] + cs * v[e]; }
    }
  }
}
template <int R>
__device__ __forceinline__ bool jacobi_pair(double* xi, double* xj, double* vi, double* vj, int m, int n, int lane) {
  double aa = 0.0, bb = 0.0, cc = 0.0;
  double u[R], v[R];
  const bool inreg = m <= 32 * R;
  for (int r0 = 0; r0 < m; r0 += 32 * R) {
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int r = r0 + lane + 32 * e;
      u[e] = r < m ? __ldcg(xi + r) : 0.0;
      v[e] = r < m ? __ldcg(xj + r) : 0.0;
    }
#pragma unroll
    for (int e = 0; e < R; ++e) {
      if (r0 + lane + 32 * e < m) { aa += u[e] * u[e]; bb += v[e] * v[e]; cc += u[e] * v[e]; }
    }
  }
  aa = warp_allsum(aa); bb = warp_allsum(bb); cc = warp_allsum(cc);
  if (cc == 0.0 || fabs(cc) <= 1e-15 * sqrt(aa * bb)) return false;
  const double zeta = (bb - aa) / (2.0 * cc);
  const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double cs = 1.0 / sqrt(1.0 + tt * tt), sn = cs * tt;
  if (inreg) {
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int r = lane + 32 * e;
      if (r < m) { xi[r] = cs * u[e] - sn * v[e]; xj[r] = sn * u[e] + cs * v[e]; }
    }
  } else {
    rot_cols<R>(xi, xj, m, lane, cs, sn);
  }
  rot_cols<R>(vi, vj, n, lane, cs, sn);
  return true;
}

// k_svdproj: one matrix of the view per cluster of `cl` CTAs (cl = 1: a
// plain launch).  The CTAs of a cluster split the column pairs of every
// round-robin round (cluster barrier between rounds), then each CTA forms
// the singular values and f / lambda redundantly and writes its share of
// the output entries.
template <class T>
__global__ void __launch_bounds__(SVD_BLOCK) k_svdproj(const __grid_constant__ Prob<T> P, int i, int which, int cl) {
  pdl_begin();
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  const bool check = (C.k % C.opt.check_every) == 0;
  if (which == 1 && !check) return;
  const Geo& g = P.g;
  const SetD<T>& S = P.set[i];
  const MatView mv = mat_view(g.ndim, g.nz_g, g.ny, g.nx, S.prim[0]);
  const int m = mv.m, n = mv.n;
  const int crank = cl > 1 ? (int)cl_rank() : 0;
  const int b = blockIdx.x / cl;
  double* X = P.svdX + (size_t)b * m * n;
  double* V = P.svdV + (size_t)b * n * n;
  const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
  constexpr int NW = SVD_BLOCK / 32;
  const int ct = crank * SVD_BLOCK + tid, cstep = cl * SVD_BLOCK;   // thread index within the cluster
  __shared__ double lam[SVD_NMAX];
  __shared__ double gsc[SVD_NMAX];
  __shared__ int s_rot[2];
  __shared__ int s_nz;
  __shared__ short s_jl[SVD_NMAX];
  __shared__ double sh[NW + 1];
  const T* src = which == 0 ? S.w : (which == 1 ? S.s : S.y[1]);
  // load: column j of X = column j of a (tr = 0) or row j of a (tr = 1)
  for (int64_t q = ct; q < (int64_t)m * n; q += cstep) {
    const int j = (int)(q / m), r = (int)(q - (int64_t)j * m);
    const int ar = mv.tr ? j : r, ac = mv.tr ? r : j;
    X[q] = (double)src[mat_pt(g, b, ar, ac)];
  }
  for (int64_t q = ct; q < (int64_t)n * n; q += cstep) V[q] = (q / n == q % n) ? 1.0 : 0.0;
  if (tid == 0) { s_rot[0] = 0; s_rot[1] = 0; }
  cl_sync(cl);
  // one-sided Jacobi sweeps, round-robin pairing of n' = n (+1 if odd) players
  const int np = n + (n & 1);
  const unsigned rot0 = cl > 1 ? cl_map(&s_rot[0], 0) : 0u;
  for (int sweep = 0; sweep < 60 && n > 1; ++sweep) {
    bool rotated = false;
    for (int t = 0; t < np - 1; ++t) {
      for (int k = crank * NW + wp; k < np / 2; k += cl * NW) {
        int a = k == 0 ? np - 1 : (t + k) % (np - 1);
        int c = (t - k + (np - 1)) % (np - 1);
        if (k == 0) c = t % (np - 1);
        if (a >= n || c >= n) continue;            // the dummy player of odd n
        const int ci = min(a, c), cj = max(a, c);
        rotated |= jacobi_pair<16>(X + (size_t)ci * m, X + (size_t)cj * m, V + (size_t)ci * n, V + (size_t)cj * n,
                                   m, n, lane);
      }
      cl_sync(cl);
    }
    // did any warp of the cluster rotate in this sweep (flag of this sweep's parity in CTA 0)
    const int par = sweep & 1;
    if (rotated && lane == 0) {
      if (cl > 1) cl_st(rot0 + 4u * par, 1);
      else s_rot[par] = 1;
    }
    cl_sync(cl);
    const int any = cl > 1 ? cl_ld(rot0 + 4u * par) : s_rot[par];
    if (crank == 0 && tid == 0) s_rot[par ^ 1] = 0;   // last read a sweep ago (all CTAs passed the barrier)
    if (!any) break;
  }
  cl_sync(cl);   // every CTA has read CTA 0's flag before any CTA can exit
  // singular values (every CTA of the cluster, the same values)
  for (int j = wp; j < n; j += NW) {
    const double* xj = X + (size_t)j * m;
    double a = 0.0;
    for (int r = lane; r < m; r += 32) { const double u = __ldcg(xj + r); a += u * u; }
    a = warp_sum(a);
    if (lane == 0) lam[j] = sqrt(a);
  }
  __syncthreads();
  if (which == 2) {   // the nuclear norm of this matrix
    double a = 0.0;
    for (int j = tid; j < n; j += SVD_BLOCK) a += lam[j];
    a = block_sum(a, sh);
    if (tid == 0) P.partials[(size_t)blockIdx.x * 4] = crank == 0 ? a : 0.0;
  } else {
    // f_j / lambda_j
    const bool rank = S.kind == K_RANK;
    double theta = 0.0;
    bool keep_all = false;
    if (!rank) {
      double tot = 0.0;
      for (int j = tid; j < n; j += SVD_BLOCK) tot += lam[j];
      tot = block_sum(tot, sh);
      const double sigma = C.sigma[i];
      keep_all = tot <= sigma;
      if (!keep_all) {
        // Duchi on the values: the active set {lambda >= lambda_j} of the
        // largest size c with lambda_j > (sum of the active - sigma) / c
        __shared__ int s_best;
        __shared__ double s_theta;
        if (tid == 0) { s_best = -1; s_theta = 0.0; }
        __syncthreads();
        for (int j = tid; j < n; j += SVD_BLOCK) {
          double sm = 0.0;
          int cnt = 0;
          for (int l = 0; l < n; ++l)
            if (lam[l] > lam[j] || (lam[l] == lam[j] && l <= j)) { sm += lam[l]; ++cnt; }
          const double th = (sm - sigma) / (double)cnt;
          if (lam[j] - th > 0.0) atomicMax(&s_best, cnt);
        }
        __syncthreads();
        for (int j = tid; j < n; j += SVD_BLOCK) {
          double sm = 0.0;
          int cnt = 0;
          for (int l = 0; l < n; ++l)
            if (lam[l] > lam[j] || (lam[l] == lam[j] && l <= j)) { sm += lam[l]; ++cnt; }
          if (cnt == s_best) s_theta = (sm - sigma) / (double)cnt;
        }
        __syncthreads();
        theta = s_theta;
        if (sigma <= 0.0) theta = INFINITY;
      }
    }
    const long long r_keep = C.kcard[i];
    for (int j = tid; j < n; j += SVD_BLOCK) {
      double f;
      if (rank) {
        int pos = 0;
        for (int l = 0; l < n; ++l) pos += (lam[l] > lam[j] || (lam[l] == lam[j] && l < j)) ? 1 : 0;
        f = pos < r_keep ? lam[j] : 0.0;
      } else {
        f = keep_all ? lam[j] : fmax(lam[j] - theta, 0.0);
      }
      gsc[j] = (lam[j] > 0.0 && f > 0.0) ? f / lam[j] : 0.0;
    }
    __syncthreads();
    if (tid == 0) {   // the columns that contribute, in index order
      int c = 0;
      for (int j = 0; j < n; ++j)
        if (gsc[j] != 0.0) s_jl[c++] = (short)j;
      s_nz = c;
    }
    __syncthreads();
    const int nz = s_nz;
    // P(a) element by element: X diag(g) V^T, mapped back to the field
    const T rho = (T)C.rho[i];
    const int par = C.k & 1;
    const bool dots = which == 0 && is_adapt_it(C.k, C.opt.adapt_every) && C.first_adapt_done;
    T* yw = S.y[par ^ 1];
    T* vw = S.v[par ^ 1];
    double a_gv = 0.0, a_gg = 0.0, a_vv = 0.0, a_fn = 0.0;
    for (int64_t q = ct; q < (int64_t)m * n; q += cstep) {
      const int c = (int)(q / m), r = (int)(q - (int64_t)c * m);   // element (r, c) of X-space
      double y = 0.0;
      for (int e = 0; e < nz; ++e) {
        const int j = s_jl[e];
        y += __ldcg(X + (size_t)j * m + r) * gsc[j] * __ldcg(V + (size_t)j * n + c);
      }
      const int ar = mv.tr ? c : r, ac = mv.tr ? r : c;
      const int64_t pt = mat_pt(g, b, ar, ac);
      if (which == 0) {
        const T wt = S.w[pt];
        const T yt = (T)y;
        const T vt = rho * (yt - wt);                 // Eq. 21 as rho (y - w), L26
        if (dots) {
          const double dg = (double)yw[pt] - (double)yt;
          const double dv = (double)vt - (double)vw[pt];
          a_gv += dg * dv; a_gg += dg * dg; a_vv += dv * dv;
        }
        yw[pt] = yt;
        vw[pt] = vt;
      } else {
        const double d = (double)S.s[pt] - (double)(T)y;
        a_fn += d * d;
      }
    }
    const double p0 = block_sum(a_gv, sh), p1 = block_sum(a_gg, sh), p2 = block_sum(a_vv, sh),
                 p3 = block_sum(a_fn, sh);
    if (tid == 0) {
      double* pp = P.partials + (size_t)blockIdx.x * 4;
      pp[0] = p0; pp[1] = p1; pp[2] = p2; pp[3] = p3;
    }
  }
  if (last_block(P.counter)) {
    __shared__ double out[4];
    for (int q = 0; q < 4; ++q) {
      double a = 0.0;
      for (int bb = tid; bb < (int)gridDim.x; bb += SVD_BLOCK) a += __ldcg(P.partials + (size_t)bb * 4 + q);
      a = block_sum(a, sh);
      if (tid == 0) out[q] = a;
    }
    __syncthreads();
    if (tid == 0) {
      *P.counter = 0u;
      if (which == 0) {
        C.sums[i][SLOT_GV] = out[0];
        C.sums[i][SLOT_GG] = out[1];
        C.sums[i][SLOT_VV] = out[2];
      } else if (which == 1) {
        C.sums[i][SLOT_FN] = out[3];
      } else {                                        // relative radius (reading L23/L29)
        C.sigma[i] = C.u_sigma[i] * out[0];
      }
    }
  }
}

}  // namespace sip
