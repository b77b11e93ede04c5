// sip_kernels.cuh -- sm_100a kernels of the PARSDMM hot path (arXiv 1902.09699).
//
// One outer iteration (Algorithm 1) is this launch sequence, all
// on one stream and captured into a CUDA graph by the runtime:
//
//   [k_blur_t]  k_rhs                       x-update right-hand side + r0
//   { [k_blur_t] k_cg1  k_cg2 } x n_cg       CG on Eq. 23, stop rule Eq. 25
//   k_pass1                                 s = A x, relaxation, pointwise
//                                           projections + duals, Alg. 2 dots,
//                                           Eq. 26/27 statistics
//   k_select x ROUNDS                       radix threshold search (l1, card)
//   k_tiecount                              index-ordered ties (cardinality)
//   k_pass2                                 global projections + duals
//   k_control                               Alg. 2, Eq. 28, coefficients
//
// Every kernel reads the device-resident Ctrl block for its decisions, so the
// captured graph is the same for every iteration.  Reductions are fixed-order
// (per-warp shuffle trees, per-CTA partials, last-CTA sum): bitwise
// reproducible for a given launch geometry.  Vectors are stored in T
// (float or double); all per-point arithmetic and every reduction is fp64
// (reading L20).
#pragma once
#include "sip_device.cuh"

namespace sip {

template <class T>
struct Prob {
  Geo g;
  int P, p;                       // p sets + distance block
  int has[NPRIM];                 // primitive present in some set
  int nglob;                      // number of global sets
  int rounds;                     // radix rounds for T
  int ntiles_pb;                  // tiles of BLOCK points per block (pass2, ties)
  SetD<T> set[MAXP];
  T* x; const T* m; T* r; T* pb[2]; T* tb;
  // deferred x update (vectorised path, n_cg <= MAXCG): p_j lives in ring
  // slot j for the whole CG solve, the CG kernels never touch x, and k_cgx
  // forms x += alpha_0 p_0 + alpha_1 p_1 + ... in that order afterwards
  // (the same fp operations, in the same order, as per-step updates)
  T* pr[MAXCG];
  int defer_x;
  T* hist[HIST_S];
  T* xs[2];
  Ctrl* ctrl;
  double* partials;               // [grid][nv]
  unsigned* counter;
  unsigned* gh_cnt;               // [MAXJOBS][NBUCK]
  unsigned long long* gh_s0;      // [MAXJOBS][NBUCK]
  unsigned long long* gh_s1;
  unsigned long long* gh_ta;      // select v2 round A: sums of key bits 19..12 per bucket [MAXJOBS][NBUCK]
  int sel_tsum;
  int selb_ns;                    // k_selB: stages of its bulk-copy ring
  unsigned* sel_gen;              // k_selCF: rounds released by the resolving CTA (only ever grows)                   // select v2: pass 1 accumulates gh_ta for l1 jobs on non-check iterations
  int* tiecnt;                    // [MAXJOBS][ntiles]
  int ntiles_max;
  // flattened segments (sip_flat.cuh): pass1 = x work + every (set, block);
  // pass2 = every (global set, block)
  int nseg1, nseg2;
  // cand[job]: keys of the radix round-1 bucket, compacted by round 2 (fp32)
  unsigned* cand[MAXJOBS];
  unsigned* ccnt;                 // [MAXJOBS][select grid]: candidates per CTA region
  long long cand_per;             // candidate region per select CTA (entries)
  int sel_grid;                   // the grid k_selectf is sized for (regions, ccnt stride)
  int p1_hint;                    // pass 1: L2 eviction hints on the staged copies (0 none, 1 x evict_last, 2 + others evict_first)
  int p1_pool, p1a_pool;          // pass 1: array slots of the bulk-copy stage pool (plain, adapt iterations)
  int p1_sub;                     // pass 1: chunks per sub-range (every segment runs over one sub-range before the next)
  int selv2;                      // single-rank fp32: round A in pass 1, k_selB / k_selC (sip_select2.cuh)
  unsigned* gf_cnt;               // select v2: k_selB's candidate histogram [MAXJOBS][256]
  unsigned long long* gf_s0;
  T* ub;                          // vectorised CG with a separable blur: c_F G^T S G p_j (sip_blur.cuh)
  double gz_[MAXTAPS / 9], gx[MAXTAPS / 9];   // the blur's separable factors, K[r][c] = gz_[r] gx[c]
  double* svdX;                   // rank / nuclear sets: fp64 Jacobi scratch, X (m x n) per matrix
  double* svdV;                   //   and V (n x n) per matrix
  int poison;                     // SIP_POISON: k_init writes NaN into fields that are written before read
  int init_zero;                  // k_init zeroes every state field (scalar kernels)
  double* fibv;                   // z slabs: this rank's fiber-set sums (4 per set), added to pass 2's
  short seg_set[64], seg_blk[64];
  short seg2_set[64], seg2_blk[64];
  double taps[MAXTAPS];           // blur kernel (row major kh x kw)
  // z-slab decomposition: with nranks > 1 the last CTA of a
  // reducing kernel publishes its rank-local values to slot `rank` of the
  // gather buffer xg (nranks slots of xslot doubles) instead of deciding;
  // the runtime exchanges the slots and k_fin (sip_team.cuh) sums them in
  // rank order and runs the same finaliser on every rank.
  int nranks, rank;
  double* xg;
  int xslot;
  FastDiv dncr;                   // division by the chunks per x row (lean CG kernels)
};

__device__ __forceinline__ bool is_adapt_it(int k, int every) {
  return every <= 1 || (k % every) == 1;   // mod(k, update-frequency) = 1
}

// ------------------------------------------------------------ finalisers
// The decision taken once the global value of a reduction is known.  One
// thread (fin_rhs / fin_cg1 / fin_cg2) or one CTA (the template ones below).

// after the rhs: ||b||^2, ||r0||^2 -> Eq. 25 target and the CG flags (L18)
__device__ inline void fin_rhs(Ctrl& C, const double* v) {
  const double bbv = v[0], rrv = v[1];
  C.bb = bbv; C.rr = rrv; C.rr_prev = rrv; C.beta = 0.0;
  C.cg_j = 0; C.cg_count = 0;
  C.zero_x = (bbv == 0.0);
  double tol = 0.0;
  if (bbv > 0.0) {
    tol = 0.1 * sqrt(rrv) / sqrt(bbv);          // Eq. 25
    if (tol < C.opt.cg_tol_floor) tol = C.opt.cg_tol_floor;
  }
  C.tol = tol;
  int active = (bbv > 0.0) && (rrv > 0.0) && (C.opt.n_cg > 0);
  if (active && C.opt.eq25 && sqrt(rrv) / sqrt(bbv) < tol) active = 0;
  C.cg_active = active;
}

// after <p_j, C p_j>: alpha, or breakdown (p.q <= 0, reading L18)
__device__ inline void fin_cg1(Ctrl& C, const double* v, int j) {
  if (v[0] > 0.0) {
    C.alpha = C.rr / v[0];
    if (j < MAXCG) C.alph[j] = C.alpha;
  } else {
    C.cg_active = 0;
    C.breakdown = 1;
  }
}

// after <r, r>: beta, Eq. 25 test, CG counters
__device__ inline void fin_cg2(Ctrl& C, const double* v, int j) {
  const double rn = v[0];
  C.beta = rn / C.rr;
  C.rr_prev = C.rr;
  C.rr = rn;
  C.cg_count += 1;
  C.cg_j = j + 1;
  int active = (C.cg_j < C.opt.n_cg) && (rn > 0.0);
  if (active && C.opt.eq25 && sqrt(rn) / sqrt(C.bb) < C.tol) active = 0;
  C.cg_active = active;
}

// p_j of the CG solve: ring slot j (deferred x) or the ping-pong pair
template <class T>
__device__ __forceinline__ T* p_slot(const Prob<T>& P, int j) {
  return P.defer_x ? P.pr[j] : P.pb[j & 1];
}

// rank-local values -> this rank's gather slot (threads of one CTA, strided)
template <class T>
__device__ __forceinline__ void publish(const Prob<T>& P, const double* v, int n, int tid, int nt) {
  double* dst = P.xg + (size_t)P.rank * P.xslot;
  for (int i = tid; i < n; i += nt) dst[i] = v[i];   // v: shared, or global written by this CTA
}

// ------------------------------------------------------------ value fetchers
template <class T>
struct VF {  // plain vector
  const T* v;
  __device__ __forceinline__ double operator()(int i) const { return (double)v[i]; }
};
template <class T>
struct PF {  // p_new = r + beta p_old, rounded to storage precision (as k_cg1 stores it)
  const T* r; const T* p; double beta; int use_p;
  __device__ __forceinline__ double operator()(int i) const {
    return use_p ? (double)(T)((double)r[i] + beta * (double)p[i]) : (double)r[i];
  }
};

// G x at a point: 'same' correlation, zero outside the grid (reading L21)
template <class F>
__device__ __forceinline__ double blur_fwd_at(const Geo& g, const double* taps, const F& f, int pt,
                                              const Loc& L) {
  const int rh = g.kh / 2, rw = g.kw / 2;
  double a = 0.0;
  for (int i = 0; i < g.kh; ++i) {
    int gz = L.gz + i - rh;
    if (gz < 0 || gz >= g.nz_g) continue;
    for (int j = 0; j < g.kw; ++j) {
      int ix = L.ix + j - rw;
      if (ix < 0 || ix >= g.nx) continue;
      a += taps[i * g.kw + j] * f(pt + (i - rh) * g.nx + (j - rw));
    }
  }
  return a;
}
// G^T u at a point: the mirrored taps
template <class F>
__device__ __forceinline__ double blur_adj_at(const Geo& g, const double* taps, const F& f, int pt,
                                              const Loc& L) {
  const int rh = g.kh / 2, rw = g.kw / 2;
  double a = 0.0;
  for (int i = 0; i < g.kh; ++i) {
    int dz = -(i - rh);
    int gz = L.gz + dz;
    if (gz < 0 || gz >= g.nz_g) continue;
    for (int j = 0; j < g.kw; ++j) {
      int dx = -(j - rw);
      int ix = L.ix + dx;
      if (ix < 0 || ix >= g.nx) continue;
      a += taps[i * g.kw + j] * f(pt + dz * g.nx + dx);
    }
  }
  return a;
}

// (A_prim x)[pt], 0 on pads (Eq. 8; F = S G, reading L21)
template <class F>
__device__ __forceinline__ double prim_fwd(const Geo& g, const double* taps, int prim, const F& f,
                                           int pt, const Loc& L) {
  switch (prim) {
    case PRIM_I: return f(pt);
    case PRIM_Z: return (L.gz < g.nz_g - 1) ? (f(pt + g.plane) - f(pt)) * g.ihz : 0.0;
    case PRIM_Y: return (L.iy < g.ny - 1) ? (f(pt + g.nx) - f(pt)) * g.ihy : 0.0;
    case PRIM_X: return (L.ix < g.nx - 1) ? (f(pt + 1) - f(pt)) * g.ihx : 0.0;
    default: return g.mask[pt] ? blur_fwd_at(g, taps, f, pt, L) : 0.0;
  }
}

// (C p)[pt] with merged coefficients: C = cI I + cz Dz'Dz + cy Dy'Dy + cx Dx'Dx
// + cF G' S' S G (Eq. 23 with Eq. 24's bookkeeping done on the scalars).
// tb = S G p (mask * G p) is precomputed by k_blur_t when F is present.
template <class T, class F>
__device__ __forceinline__ double apply_C_at(const Prob<T>& P, const Ctrl& C, const F& f, int pt,
                                             const Loc& L) {
  const Geo& g = P.g;
  const double p0 = f(pt);
  double q = C.cI * p0;
  if (P.has[PRIM_Z]) {
    double a = 0.0;
    if (L.gz >= 1) a += p0 - f(pt - g.plane);
    if (L.gz < g.nz_g - 1) a -= f(pt + g.plane) - p0;
    q += C.cz * a;
  }
  if (P.has[PRIM_Y]) {
    double a = 0.0;
    if (L.iy >= 1) a += p0 - f(pt - g.nx);
    if (L.iy < g.ny - 1) a -= f(pt + g.nx) - p0;
    q += C.cy * a;
  }
  if (P.has[PRIM_X]) {
    double a = 0.0;
    if (L.ix >= 1) a += p0 - f(pt - 1);
    if (L.ix < g.nx - 1) a -= f(pt + 1) - p0;
    q += C.cx * a;
  }
  if (P.has[PRIM_F]) q += C.cF * blur_adj_at(g, P.taps, VF<T>{P.tb}, pt, L);
  return q;
}

// ------------------------------------------------------------ per-warp accumulation
__device__ __forceinline__ void warp_acc(double* acc, int nv, int slot, double v) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) acc[(threadIdx.x >> 5) * nv + slot] += v;
}

// sum the per-warp accumulators, write the CTA partials, last CTA reduces into out[]
__device__ inline bool finish_reduction(double* acc, int nv, double* partials, unsigned* counter,
                                        double* out, double* sh) {
  __syncthreads();
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double a = 0.0;
    for (int w = 0; w < NWARP; ++w) a += acc[w * nv + v];
    partials[(size_t)blockIdx.x * nv + v] = a;
  }
  bool last = last_block(counter);
  if (last) {
    reduce_partials(partials, nv, out, sh);
    if (threadIdx.x == 0) *counter = 0u;
  }
  return last;
}

// ------------------------------------------------------------ k_blur_t
// tb = mask * G(src); mode 0: src = x, mode 1: src = r + beta p (CG step j)
template <class T>
__global__ void __launch_bounds__(BLOCK) k_blur_t(const __grid_constant__ Prob<T> P, int mode, int j) {
  const Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  if (mode == 1 && !C.cg_active) return;
  const Geo& g = P.g;
  PF<T> pf{P.r, P.pb[(j + 1) & 1], C.beta, j > 0};
  for (int pt = blockIdx.x * BLOCK + threadIdx.x; pt < g.N; pt += gridDim.x * BLOCK) {
    Loc L = locate(g, pt);
    double t = 0.0;
    if (g.mask[pt]) t = (mode == 0) ? blur_fwd_at(g, P.taps, VF<T>{P.x}, pt, L)
                                    : blur_fwd_at(g, P.taps, pf, pt, L);
    P.tb[pt] = (T)t;
  }
}

// ------------------------------------------------------------ k_rhs
// b = sum_i A_i^T (rho_i y_i + v_i)  (Eq. 21 line 1), r = b - C x^k,
// ||b||^2, ||r||^2; last CTA sets the Eq. 25 target and the CG flags.
template <class T>
__global__ void __launch_bounds__(BLOCK) k_rhs(const __grid_constant__ Prob<T> P) {
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  __shared__ double sh[NWARP + 1];
  __shared__ double out[2];
  const Geo& g = P.g;
  const int par = C.k & 1;
  double bb = 0.0, rr = 0.0;
  for (int pt = blockIdx.x * BLOCK + threadIdx.x; pt < g.N; pt += gridDim.x * BLOCK) {
    Loc L = locate(g, pt);
    double b = 0.0;
    for (int i = 0; i < P.P; ++i) {
      const SetD<T>& S = P.set[i];
      const double rho = C.rho[i];
      const T* y = S.y[par];
      const T* v = S.v[par];
      for (int bl = 0; bl < S.nblk; ++bl) {
        const int64_t o = (int64_t)bl * g.ld;
        auto u = [&](int q) { return rho * (double)y[o + q] + (double)v[o + q]; };
        switch (S.prim[bl]) {
          case PRIM_I: b += u(pt); break;
          case PRIM_Z: {  // D_z^T: +u[z-1] - u[z] (pads hold 0)
            double a = 0.0;
            if (L.gz >= 1) a += u(pt - g.plane);
            if (L.gz < g.nz_g - 1) a -= u(pt);
            b += a * g.ihz;
            break;
          }
          case PRIM_Y: {
            double a = 0.0;
            if (L.iy >= 1) a += u(pt - g.nx);
            if (L.iy < g.ny - 1) a -= u(pt);
            b += a * g.ihy;
            break;
          }
          case PRIM_X: {
            double a = 0.0;
            if (L.ix >= 1) a += u(pt - 1);
            if (L.ix < g.nx - 1) a -= u(pt);
            b += a * g.ihx;
            break;
          }
          default: {  // F^T u = G^T (S^T u); u is zero off the mask
            struct UF { const T* y; const T* v; double rho; __device__ double operator()(int q) const {
              return rho * (double)y[q] + (double)v[q]; } } uf{y + o, v + o, rho};
            b += blur_adj_at(g, P.taps, uf, pt, L);
          }
        }
      }
    }
    double cx = apply_C_at(P, C, VF<T>{P.x}, pt, L);
    T rt = (T)(b - cx);
    P.r[pt] = rt;
    bb += b * b;
    rr += (double)rt * (double)rt;
  }
  bb = block_sum(bb, sh);
  rr = block_sum(rr, sh);
  double* part = P.partials;
  if (threadIdx.x == 0) { part[blockIdx.x * 2] = bb; part[blockIdx.x * 2 + 1] = rr; }
  if (last_block(P.counter)) {
    reduce_partials(part, 2, out, sh);
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      const double bbv = out[0], rrv = out[1];
      C.bb = bbv; C.rr = rrv; C.rr_prev = rrv; C.beta = 0.0;
      C.cg_j = 0; C.cg_count = 0;
      C.zero_x = (bbv == 0.0);
      double tol = 0.0;
      if (bbv > 0.0) {
        tol = 0.1 * sqrt(rrv) / sqrt(bbv);          // Eq. 25
        if (tol < C.opt.cg_tol_floor) tol = C.opt.cg_tol_floor;
      }
      C.tol = tol;
      int active = (bbv > 0.0) && (rrv > 0.0) && (C.opt.n_cg > 0);
      if (active && C.opt.eq25 && sqrt(rrv) / sqrt(bbv) < tol) active = 0;
      C.cg_active = active;
    }
  }
}

// ------------------------------------------------------------ CG (Hestenes-Stiefel)
// k_cg1(j): p_j = r + beta p_{j-1} (p_0 = r), q = C p_j, <p_j, q>; alpha
template <class T>
__global__ void __launch_bounds__(BLOCK) k_cg1(const __grid_constant__ Prob<T> P, int j) {
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  const Geo& g = P.g;
  if (j == 0 && C.zero_x) {   // b = 0 gives x = 0
    for (int pt = blockIdx.x * BLOCK + threadIdx.x; pt < g.N; pt += gridDim.x * BLOCK) P.x[pt] = (T)0;
    return;
  }
  if (!C.cg_active) return;
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  PF<T> pf{P.r, P.pb[(j + 1) & 1], C.beta, j > 0};
  T* pw = P.pb[j & 1];
  double pq = 0.0;
  for (int pt = blockIdx.x * BLOCK + threadIdx.x; pt < g.N; pt += gridDim.x * BLOCK) {
    Loc L = locate(g, pt);
    double p0 = pf(pt);
    pw[pt] = (T)p0;
    double q = apply_C_at(P, C, pf, pt, L);
    pq += p0 * q;
  }
  pq = block_sum(pq, sh);
  if (threadIdx.x == 0) P.partials[blockIdx.x] = pq;
  if (last_block(P.counter)) {
    reduce_partials(P.partials, 1, out, sh);
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      if (out[0] > 0.0) {
        C.alpha = C.rr / out[0];
      } else {               // breakdown: p.q <= 0 (reading L18)
        C.cg_active = 0;
        C.breakdown = 1;
      }
    }
  }
}

// k_cg2(j): x += alpha p, r -= alpha C p, <r, r>; beta, Eq. 25 test
template <class T>
__global__ void __launch_bounds__(BLOCK) k_cg2(const __grid_constant__ Prob<T> P, int j) {
  Ctrl& C = *P.ctrl;
  if (C.stopped || !C.cg_active) return;
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  const Geo& g = P.g;
  const T* pv = P.pb[j & 1];
  const double alpha = C.alpha;
  double rr = 0.0;
  for (int pt = blockIdx.x * BLOCK + threadIdx.x; pt < g.N; pt += gridDim.x * BLOCK) {
    Loc L = locate(g, pt);
    double p0 = (double)pv[pt];
    double q = apply_C_at(P, C, VF<T>{pv}, pt, L);
    P.x[pt] = (T)((double)P.x[pt] + alpha * p0);
    T rn = (T)((double)P.r[pt] - alpha * q);
    P.r[pt] = rn;
    rr += (double)rn * (double)rn;
  }
  rr = block_sum(rr, sh);
  if (threadIdx.x == 0) P.partials[blockIdx.x] = rr;
  if (last_block(P.counter)) {
    reduce_partials(P.partials, 1, out, sh);
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      const double rn = out[0];
      C.beta = rn / C.rr;
      C.rr_prev = C.rr;
      C.rr = rn;
      C.cg_count += 1;
      C.cg_j = j + 1;
      int active = (C.cg_j < C.opt.n_cg) && (rn > 0.0);
      if (active && C.opt.eq25 && sqrt(rn) / sqrt(C.bb) < C.tol) active = 0;
      C.cg_active = active;
    }
  }
}

// ------------------------------------------------------------ k_pass1
// Algorithm 1 FOR-loop body for every set at once:
//   s_i = A_i x, x-bar = gamma s + (1-gamma) y, w = x-bar - v/rho,
//   pointwise sets: y = P(w) (box clamp / Eq. 22), v = v + rho (y - x-bar);
//   global sets: store w (projection finished in k_pass2).
// Plus Alg. 2's v-hat (old y, v; reading L10) and alpha-side dots, the
// beta-side dots of pointwise sets, Eq. 26/27 statistics, the x history.
template <class T>
__global__ void __launch_bounds__(BLOCK) k_pass1(const __grid_constant__ Prob<T> P) {
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  extern __shared__ double acc[];
  __shared__ double sh[NWARP + 1];
  const Geo& g = P.g;
  const int nv = P.P * NSLOT + NEVOL;
  const int k = C.k, par = k & 1;
  const bool adapt = is_adapt_it(k, C.opt.adapt_every);
  const bool dots = adapt && C.first_adapt_done;
  const bool check = (k % C.opt.check_every) == 0;
  const int a = C.adapt_calls;
  const T* xs_rd = P.xs[(a + 1) & 1];
  T* xs_wr = P.xs[a & 1];
  const int hcount = C.hist_count, hhead = C.hist_head;
  const int hslot = (hhead + 1) % HIST_S;
  for (int v = threadIdx.x; v < NWARP * nv; v += BLOCK) acc[v] = 0.0;
  __syncthreads();

  const int ntile = (g.N + BLOCK - 1) / BLOCK;
  for (int tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int pt = tile * BLOCK + threadIdx.x;
    const bool valid = pt < g.N;
    Loc L{0, 0, 0, 0};
    double x0 = 0.0;
    if (valid) { L = locate(g, pt); x0 = (double)P.x[pt]; }
    // Eq. 27 history norms, before the oldest slot is overwritten
    if (check) {
      warp_acc(acc, nv, P.P * NSLOT + 0, x0 * x0);
      for (int jj = 0; jj < hcount; ++jj) {
        int js = (hhead - jj + HIST_S) % HIST_S;
        double d = valid ? x0 - (double)P.hist[js][pt] : 0.0;
        warp_acc(acc, nv, P.P * NSLOT + 1 + js, d * d);
      }
    }
    if (valid) P.hist[hslot][pt] = (T)x0;
    // s = A_prim x for the primitives present; ds = A_prim (x - x^{k0})
    double s[NPRIM], ds[NPRIM];
#pragma unroll
    for (int q = 0; q < NPRIM; ++q) { s[q] = 0.0; ds[q] = 0.0; }
    if (valid) {
#pragma unroll
      for (int q = 0; q < NPRIM; ++q) {
        if (!P.has[q]) continue;
        s[q] = prim_fwd(g, P.taps, q, VF<T>{P.x}, pt, L);
        if (dots) ds[q] = s[q] - prim_fwd(g, P.taps, q, VF<T>{xs_rd}, pt, L);
      }
      if (adapt) xs_wr[pt] = (T)x0;
    }
    for (int i = 0; i < P.P; ++i) {
      const SetD<T>& S = P.set[i];
      const double rho = C.rho[i], gam = C.gamma[i];
      const T* yr = S.y[par];
      const T* vr = S.v[par];
      T* yw = S.y[par ^ 1];
      T* vw = S.v[par ^ 1];
      const bool pointwise = (S.kind == K_BOUNDS || S.kind == K_DIST);
      double a_w2 = 0, a_hv = 0, a_hh = 0, a_vh = 0, a_gv = 0, a_gg = 0, a_vv = 0, a_fn = 0, a_s2 = 0;
      for (int bl = 0; bl < S.nblk; ++bl) {
        const int prim = S.prim[bl];
        if (!valid || is_pad(g, prim, L, pt)) continue;
        const int64_t off = (int64_t)bl * g.ld + pt;
        const double sv = s[prim];
        const double yo = (double)yr[off], vo = (double)vr[off];
        const double xbar = gam * sv + (1.0 - gam) * yo;       // relaxation
        const double w = (double)(T)(xbar - vo / rho);          // as stored for global sets
        if (pointwise) {
          double yn;
          if (S.kind == K_DIST) {
            yn = ((double)P.m[pt] + rho * w) / (1.0 + rho);   // Eq. 22
          } else {
            const double lo = S.lo_vec ? (double)S.lo_vec[off] : S.lo;
            const double hi = S.hi_vec ? (double)S.hi_vec[off] : S.hi;
            yn = w < lo ? lo : (w > hi ? hi : w);
            if (check) {
              const double c = sv < lo ? lo : (sv > hi ? hi : sv);
              a_fn += (sv - c) * (sv - c);
            }
          }
          const T ynt = (T)yn;
          const T vnt = (T)(rho * ((double)ynt - w));   // Eq. 21 dual update as rho (y - w), L26
          if (dots) {
            const double dg = -((double)ynt - (double)yw[off]);
            const double dv = (double)vnt - (double)vw[off];
            a_gv += dg * dv; a_gg += dg * dg; a_vv += dv * dv;
          }
          yw[off] = ynt;
          vw[off] = vnt;
        } else {
          const T wt = (T)w;
          S.w[off] = wt;
          a_w2 += (double)wt * (double)wt;
          if (check && S.s) S.s[off] = (T)sv;
        }
        if (adapt) {                                   // Alg. 2 line 1
          const T vht = (T)(vo + rho * (yo - sv));
          if (dots) {
            const double dvh = (double)vht - (double)S.vh0[off];
            const double dh = ds[prim];
            a_hv += dh * dvh; a_hh += dh * dh; a_vh += dvh * dvh;
          }
          S.vh0[off] = vht;
        }
        if (check) a_s2 += sv * sv;
      }
      const int base = i * NSLOT;
      if (S.kind == K_L2 || S.kind == K_ANN) warp_acc(acc, nv, base + SLOT_W2, a_w2);
      if (dots) {
        warp_acc(acc, nv, base + SLOT_HV, a_hv);
        warp_acc(acc, nv, base + SLOT_HH, a_hh);
        warp_acc(acc, nv, base + SLOT_VHVH, a_vh);
        if (pointwise) {
          warp_acc(acc, nv, base + SLOT_GV, a_gv);
          warp_acc(acc, nv, base + SLOT_GG, a_gg);
          warp_acc(acc, nv, base + SLOT_VV, a_vv);
        }
      }
      if (check) {
        if (S.kind == K_BOUNDS) warp_acc(acc, nv, base + SLOT_FN, a_fn);
        warp_acc(acc, nv, base + SLOT_S2, a_s2);
      }
    }
  }
  // the sums land in C.sums / C.evol (contiguous: sums[MAXP][NSLOT] then evol
  // are not contiguous for P < MAXP, so reduce into a staging area first)
  double* stage = P.partials + (size_t)gridDim.x * nv;   // nv doubles after the partials
  if (finish_reduction(acc, nv, P.partials, P.counter, stage, sh)) {
    for (int v = threadIdx.x; v < nv; v += BLOCK) {
      double val = __ldcg(stage + v);
      if (v < P.P * NSLOT) C.sums[v / NSLOT][v % NSLOT] = val;
      else C.evol[v - P.P * NSLOT] = val;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // annulus / l2 radial factors (Table 1 rows l2, annulus; reading L7)
      for (int i = 0; i < P.P; ++i) {
        const int kd = P.set[i].kind;
        if (kd != K_L2 && kd != K_ANN) continue;
        const double n = sqrt(__ldcg(stage + i * NSLOT + SLOT_W2));
        double f = 1.0;
        int z = 0;
        if (n == 0.0) z = (C.sig_lo[i] > 0.0);
        else if (n > C.sig_hi[i]) f = C.sig_hi[i] / n;
        else if (n < C.sig_lo[i]) f = C.sig_lo[i] / n;
        C.ann_scale[i] = f;
        C.ann_zero[i] = z;
      }
    }
  }
}

// ------------------------------------------------------------ k_select
// One radix round of the threshold search (l1 ball, Duchi-equivalent exact
// theta; cardinality: exact k-th key).  Buckets hold the count and the exact
// integer sum of significands of |value| (all values of a bucket share the
// exponent), so the histograms are exact and order independent.
template <class T>
__device__ void resolve_round(const Prob<T>& P, Job& J, int round, const unsigned* hc,
                              const unsigned long long* h0, const unsigned long long* h1) {
  using K = KeyT<T>;
  using U = typename K::U;
  __shared__ long long s_cnt[BLOCK];
  __shared__ double s_sum[BLOCK];
  __shared__ int s_best[BLOCK];
  int lo, nb;
  digit_bits(K::BITS, round, &lo, &nb);
  const int nbk = 1 << nb;
  const int per = (nbk + BLOCK - 1) / BLOCK;
  const int d0 = threadIdx.x * per;
  long long c_loc = 0;
  double s_loc = 0.0;
  for (int d = d0; d < d0 + per && d < nbk; ++d) {
    c_loc += __ldcg(hc + d);
    U kb = (U)(((U)J.prefix << nb) | (U)d) << lo;
    s_loc += ((double)__ldcg(h1 + d) * 4294967296.0 + (double)__ldcg(h0 + d)) * SigT<T>::scale(kb);
  }
  s_cnt[threadIdx.x] = c_loc;
  s_sum[threadIdx.x] = s_loc;
  __syncthreads();
  if (threadIdx.x == 0) {    // suffix totals of the threads above, fixed order
    long long c = 0; double s = 0.0;
    for (int t = BLOCK - 1; t >= 0; --t) {
      long long ct = s_cnt[t]; double st = s_sum[t];
      s_cnt[t] = c; s_sum[t] = s;
      c += ct; s += st;
    }
  }
  __syncthreads();
  // walk my buckets from the top: C(>=d), S(>=d)
  long long c_ge = J.cnt_above + s_cnt[threadIdx.x];
  double s_ge = J.sum_above + s_sum[threadIdx.x];
  int best = -1;
  for (int d = min(d0 + per, nbk) - 1; d >= d0; --d) {
    U kb = (U)(((U)J.prefix << nb) | (U)d) << lo;
    c_ge += __ldcg(hc + d);
    s_ge += ((double)__ldcg(h1 + d) * 4294967296.0 + (double)__ldcg(h0 + d)) * SigT<T>::scale(kb);
    bool ok;
    if (J.kind == K_L1) ok = (s_ge - (double)K::val(kb) * (double)c_ge) > J.sigma;  // f(e_d) > sigma
    else ok = c_ge >= J.k;                                                        // C(>=d) >= k
    if (ok && d > best) best = d;
  }
  s_best[threadIdx.x] = best;
  __syncthreads();
  __shared__ int s_dstar;
  if (threadIdx.x == 0) {
    int b = -1;
    for (int t = 0; t < BLOCK; ++t) b = max(b, s_best[t]);
    s_dstar = b;
  }
  __syncthreads();
  const int dstar = s_dstar;
  // the owner of d* forms the totals strictly above d*; thread 0 the grand total
  __shared__ long long s_cab, s_ctot;
  __shared__ double s_sab, s_stot;
  if (threadIdx.x == 0) {
    s_ctot = J.cnt_above + s_cnt[0] + c_loc;
    s_stot = J.sum_above + s_sum[0] + s_loc;
  }
  if (dstar >= d0 && dstar < d0 + per) {
    long long c = J.cnt_above + s_cnt[threadIdx.x];
    double sm = J.sum_above + s_sum[threadIdx.x];
    for (int d = min(d0 + per, nbk) - 1; d > dstar; --d) {
      U kb = (U)(((U)J.prefix << nb) | (U)d) << lo;
      c += __ldcg(hc + d);
      sm += ((double)__ldcg(h1 + d) * 4294967296.0 + (double)__ldcg(h0 + d)) * SigT<T>::scale(kb);
    }
    s_cab = c;
    s_sab = sm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (J.kind == K_L1 && round == 1 && s_stot <= J.sigma) {
      J.mode = JM_INSIDE;          // ||w||_1 <= sigma: w is in the ball (L5)
    } else if (J.kind == K_L1 && round == 1 && J.sigma <= 0.0) {
      J.mode = JM_ZERO;            // sigma = 0: the ball is {0}
    } else if (dstar < 0) {
      J.mode = JM_ALL;             // not reachable for a consistent search
    } else {
      J.cnt_above = s_cab;
      J.sum_above = s_sab;
      J.prefix = (J.prefix << nb) | (unsigned long long)dstar;
      J.round = round;
      if (round == K::ROUNDS) {
        if (J.kind == K_L1) {      // entries == prefix value are inactive
          J.theta = (J.sum_above - J.sigma) / (double)J.cnt_above;
          J.mode = JM_DONE;
        } else {
          J.tau = J.prefix;
          const long long ceq = __ldcg(hc + dstar);
          J.cnt_eq = ceq;
          J.keep_eq = J.k - J.cnt_above;
          J.ties = (J.keep_eq < ceq) ? 1 : 0;
          const double tv = (double)K::val((U)J.tau);
          J.tau_val2 = tv * tv;
          J.mode = (J.tau == 0ull) ? JM_ALL : JM_DONE;
        }
      }
    }
  }
  __syncthreads();
}

template <class T>
__global__ void __launch_bounds__(BLOCK) k_select(const __grid_constant__ Prob<T> P, int round) {
  using K = KeyT<T>;
  using U = typename K::U;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  __shared__ unsigned h_cnt[NBUCK];
  __shared__ unsigned long long h_s0[NBUCK];
  __shared__ unsigned long long h_s1[NBUCK];
  const Geo& g = P.g;
  const bool check = (C.k % C.opt.check_every) == 0;
  int lo, nb, plo = 0, pnb = 0;
  digit_bits(K::BITS, round, &lo, &nb);
  if (round > 1) digit_bits(K::BITS, round - 1, &plo, &pnb);
  const U dmask = (U)((1u << nb) - 1u);
  bool any = false;
  for (int jb = 0; jb < C.njobs; ++jb) {
    const Job& J = C.job[jb];
    if (J.mode != JM_SEARCH || J.round != round - 1 || (J.on_s && !check)) continue;
    any = true;
    for (int d = threadIdx.x; d < NBUCK; d += BLOCK) { h_cnt[d] = 0u; h_s0[d] = 0ull; h_s1[d] = 0ull; }
    __syncthreads();
    const SetD<T>& S = P.set[J.set];
    const T* buf = J.on_s ? S.s : S.w;
    const U prefix = (U)J.prefix;
    const bool sums = (J.kind == K_L1);
    for (int bl = 0; bl < S.nblk; ++bl) {
      const T* bp = buf + (int64_t)bl * g.ld;
      for (int pt = blockIdx.x * BLOCK + threadIdx.x; pt < g.N; pt += gridDim.x * BLOCK) {
        const U key = K::key(bp[pt]);
        if (round > 1 && (U)(key >> plo) != prefix) continue;
        const int d = (int)((key >> lo) & dmask);
        atomicAdd(&h_cnt[d], 1u);
        if (sums) {
          unsigned long long sh_, sl_;
          SigT<T>::split(key, &sh_, &sl_);
          atomicAdd(&h_s0[d], sl_);
          if (sh_) atomicAdd(&h_s1[d], sh_);
        }
      }
    }
    __syncthreads();
    unsigned* gc = P.gh_cnt + (size_t)jb * NBUCK;
    unsigned long long* g0 = P.gh_s0 + (size_t)jb * NBUCK;
    unsigned long long* g1 = P.gh_s1 + (size_t)jb * NBUCK;
    for (int d = threadIdx.x; d < (1 << nb); d += BLOCK) {
      if (h_cnt[d]) atomicAdd(gc + d, h_cnt[d]);
      if (h_s0[d]) atomicAdd(g0 + d, h_s0[d]);
      if (h_s1[d]) atomicAdd(g1 + d, h_s1[d]);
    }
    __syncthreads();
  }
  if (!any) return;
  if (last_block(P.counter)) {
    for (int jb = 0; jb < C.njobs; ++jb) {
      Job& J = C.job[jb];
      if (J.mode != JM_SEARCH || J.round != round - 1 || (J.on_s && !check)) continue;
      unsigned* gc = P.gh_cnt + (size_t)jb * NBUCK;
      unsigned long long* g0 = P.gh_s0 + (size_t)jb * NBUCK;
      unsigned long long* g1 = P.gh_s1 + (size_t)jb * NBUCK;
      resolve_round<T>(P, J, round, gc, g0, g1);
      for (int d = threadIdx.x; d < NBUCK; d += BLOCK) { gc[d] = 0u; g0[d] = 0ull; g1[d] = 0ull; }
      __syncthreads();
    }
    if (threadIdx.x == 0) *P.counter = 0u;
  }
}

// ------------------------------------------------------------ k_tiecount
// cardinality ties at tau: per-tile counts, then exclusive scan in tile order
// (= global index order, reading L6)
template <class T>
__global__ void __launch_bounds__(BLOCK) k_tiecount(const __grid_constant__ Prob<T> P) {
  using K = KeyT<T>;
  using U = typename K::U;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  __shared__ int s_w[NWARP];
  __shared__ long long s_c[BLOCK];
  const Geo& g = P.g;
  bool any = false;
  for (int i = 0; i < P.P; ++i) {
    const SetD<T>& S = P.set[i];
    if (S.kind != K_CARD) continue;
    const Job& J = C.job[S.job];
    if (J.mode != JM_DONE || !J.ties) continue;
    any = true;
    int* tc = P.tiecnt + (size_t)S.job * P.ntiles_max;
    const int nt = S.nblk * P.ntiles_pb;
    for (int t = blockIdx.x; t < nt; t += gridDim.x) {
      const int bl = t / P.ntiles_pb, lt = t - bl * P.ntiles_pb;
      const int pt = lt * BLOCK + threadIdx.x;
      bool f = false;
      if (pt < g.N) f = (K::key(S.w[(int64_t)bl * g.ld + pt]) == (U)J.tau);
      unsigned bal = __ballot_sync(0xffffffffu, f);
      if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = __popc(bal);
      __syncthreads();
      if (threadIdx.x == 0) {
        int c = 0;
        for (int w = 0; w < NWARP; ++w) c += s_w[w];
        tc[t] = c;
      }
      __syncthreads();
    }
  }
  if (!any) return;
  if (last_block(P.counter)) {
    for (int i = 0; i < P.P; ++i) {
      const SetD<T>& S = P.set[i];
      if (S.kind != K_CARD) continue;
      const Job& J = C.job[S.job];
      if (J.mode != JM_DONE || !J.ties) continue;
      int* tc = P.tiecnt + (size_t)S.job * P.ntiles_max;
      const int nt = S.nblk * P.ntiles_pb;
      const int per = (nt + BLOCK - 1) / BLOCK;
      const int t0 = threadIdx.x * per;
      long long loc = 0;
      for (int t = t0; t < t0 + per && t < nt; ++t) loc += __ldcg(tc + t);
      s_c[threadIdx.x] = loc;
      __syncthreads();
      if (threadIdx.x == 0) {
        long long run = 0;
        for (int t = 0; t < BLOCK; ++t) { long long c = s_c[t]; s_c[t] = run; run += c; }
      }
      __syncthreads();
      long long run = s_c[threadIdx.x];
      for (int t = t0; t < t0 + per && t < nt; ++t) {
        int c = __ldcg(tc + t);
        tc[t] = (int)run;           // exclusive offset of tile t
        run += c;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) *P.counter = 0u;
  }
}

// ------------------------------------------------------------ k_pass2
// Global sets: y = P_C(w) with the resolved theta / tau / radial factor,
// v = rho (y - w)  (= v + rho (y - x-bar), Eq. 21), Alg. 2 beta-side dots.
// Check iterations: Eq. 26 numerators of l1 / cardinality sets from s.
template <class T>
__global__ void __launch_bounds__(BLOCK) k_pass2(const __grid_constant__ Prob<T> P) {
  using K = KeyT<T>;
  using U = typename K::U;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  extern __shared__ double acc[];
  __shared__ double sh[NWARP + 1];
  __shared__ int s_w[NWARP];
  const Geo& g = P.g;
  const int nv = P.P * 4;     // per set: gv, gg, vv, fn
  const int k = C.k, par = k & 1;
  const bool adapt = is_adapt_it(k, C.opt.adapt_every);
  const bool dots = adapt && C.first_adapt_done;
  const bool check = (k % C.opt.check_every) == 0;
  for (int v = threadIdx.x; v < NWARP * nv; v += BLOCK) acc[v] = 0.0;
  __syncthreads();
  for (int i = 0; i < P.P; ++i) {
    const SetD<T>& S = P.set[i];
    if (!S.global || S.svd) continue;
    const double rho = C.rho[i];
    const Job* J = (S.kind == K_L1 || S.kind == K_CARD) ? &C.job[S.job] : nullptr;
    const int mode = J ? J->mode : JM_DONE;
    const double theta = J ? J->theta : 0.0;
    const U tau = J ? (U)J->tau : (U)0;
    const long long keep_eq = J ? J->keep_eq : 0;
    const int ties = J ? J->ties : 0;
    const double scale = C.ann_scale[i];
    const int azero = C.ann_zero[i];
    const int* toff = (S.kind == K_CARD) ? P.tiecnt + (size_t)S.job * P.ntiles_max : nullptr;
    T* yw = S.y[par ^ 1];
    T* vw = S.v[par ^ 1];
    double a_gv = 0, a_gg = 0, a_vv = 0;
    unsigned long long hsum = 0;   // support fingerprint (cardinality)
    const int nt = S.nblk * P.ntiles_pb;
    for (int t = blockIdx.x; t < nt; t += gridDim.x) {
      const int bl = t / P.ntiles_pb, lt = t - bl * P.ntiles_pb;
      const int pt = lt * BLOCK + threadIdx.x;
      bool valid = pt < g.N;
      Loc L{0, 0, 0, 0};
      if (valid) { L = locate(g, pt); valid = !is_pad(g, S.prim[bl], L, pt); }
      const int64_t off = (int64_t)bl * g.ld + pt;
      const double w = valid ? (double)S.w[off] : 0.0;
      double y = 0.0;
      if (S.kind == K_L1) {
        if (mode == JM_INSIDE || mode == JM_ALL) y = w;
        else if (mode == JM_DONE) {
          const double a = fabs(w) - theta;
          y = a > 0.0 ? (w > 0.0 ? a : -a) : 0.0;   // soft threshold
        }
      } else if (S.kind == K_CARD) {
        const U key = valid ? K::key((T)w) : (U)0;
        bool keep = (mode == JM_ALL);
        if (mode == JM_DONE) {
          keep = key > tau;
          if (ties) {  // keep the first keep_eq entries == tau in index order
            const bool f = valid && key == tau;
            unsigned bal = __ballot_sync(0xffffffffu, f);
            const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
            if (lane == 0) s_w[wp] = __popc(bal);
            __syncthreads();
            int before = 0;
            for (int q = 0; q < wp; ++q) before += s_w[q];
            before += __popc(bal & ((1u << lane) - 1u));
            const long long rank = (long long)toff[t] + before;
            if (f && rank < keep_eq) keep = true;
            __syncthreads();
          } else if (key == tau) {
            keep = true;
          }
        }
        y = keep ? w : 0.0;
        if (valid && y != 0.0)
          hsum += supp_mix((unsigned long long)bl * ((unsigned long long)g.nz_g * g.plane) +
                           (unsigned long long)g.z0 * g.plane + (unsigned long long)pt);
      } else {   // l2 ball / annulus: radial scaling (L7 at 0)
        y = azero ? ((bl == 0 && pt == S.first_real) ? C.sig_lo[i] : 0.0) : w * scale;
      }
      if (valid) {
        const T yt = (T)y;
        const T vt = (T)(rho * ((double)yt - w));
        if (dots) {
          const double dg = -((double)yt - (double)yw[off]);
          const double dv = (double)vt - (double)vw[off];
          a_gv += dg * dv; a_gg += dg * dg; a_vv += dv * dv;
        }
        yw[off] = yt;
        vw[off] = vt;
      }
    }
    if (dots) {
      warp_acc(acc, nv, i * 4 + 0, a_gv);
      warp_acc(acc, nv, i * 4 + 1, a_gg);
      warp_acc(acc, nv, i * 4 + 2, a_vv);
    }
    if (S.kind == K_CARD) supp_add_warp(C, i, hsum);
    // Eq. 26 numerator for l1 / cardinality from s (check iterations)
    if (check && S.sjob >= 0) {
      const Job& Js = C.job[S.sjob];
      double fn = 0.0;
      if (Js.mode == JM_DONE) {
        for (int bl = 0; bl < S.nblk; ++bl) {
          const T* sp = S.s + (int64_t)bl * g.ld;
          for (int pt = blockIdx.x * BLOCK + threadIdx.x; pt < g.N; pt += gridDim.x * BLOCK) {
            const double sv = (double)sp[pt];
            if (S.kind == K_L1) {
              const double a = fabs(sv) < Js.theta ? fabs(sv) : Js.theta;
              fn += a * a;
            } else if (K::key(sp[pt]) < (U)Js.tau) {
              fn += sv * sv;
            }
          }
        }
      }
      warp_acc(acc, nv, i * 4 + 3, fn);
    }
  }
  double* stage = P.partials + (size_t)gridDim.x * nv;
  if (finish_reduction(acc, nv, P.partials, P.counter, stage, sh)) {
    for (int v = threadIdx.x; v < nv; v += BLOCK) {
      const int i = v / 4, q = v % 4;
      if (!P.set[i].global) continue;
      const double val = __ldcg(stage + v);
      if (q == 0) C.sums[i][SLOT_GV] = val;
      if (q == 1) C.sums[i][SLOT_GG] = val;
      if (q == 2) C.sums[i][SLOT_VV] = val;
      if (q == 3 && P.set[i].sjob >= 0) C.sums[i][SLOT_FN] = val;
    }
  }
}

// ------------------------------------------------------------ control
// Algorithm 2 on the device.  Both halves of the algorithm are
// the same safeguarded spectral step applied to a pair of difference vectors
// (alpha: Delta h, Delta v_hat; beta: Delta g, Delta v), so it is written once:
// from the cross product and the two squared norms, the correlation test
// (eps_corr; a zero norm fails it, reading L17), then the
// minimum-gradient step MG = cross / |d|^2 or the steepest-descent step
// SD = |v|^2 / cross.
struct SpecStep {
  bool ok;
  double step;
};
__device__ __forceinline__ SpecStep spectral_step(double cross, double dd, double vv, double eps_corr) {
  SpecStep r{false, 0.0};
  if (!(dd > 0.0 && vv > 0.0)) return r;
  if (!(cross / (sqrt(dd) * sqrt(vv)) > eps_corr)) return r;
  const double mg = cross / dd;
  const double sd = vv / cross;
  r.ok = true;
  r.step = (2.0 * mg > sd) ? mg : sd - 0.5 * mg;
  return r;
}
// the four-way table of: branch code 0 both, 1 alpha, 2 beta, 3 none
__device__ inline int alg2_table(const SpecStep& a, const SpecStep& b, double rho, double* rho_new,
                                 double* gamma_new) {
  if (a.ok && b.ok) {
    const double g = sqrt(a.step * b.step);          // rho = sqrt(alpha_hat beta_hat)
    *rho_new = g;
    *gamma_new = 1.0 + 2.0 * g / (a.step + b.step);
    return 0;
  }
  if (!a.ok && !b.ok) {
    *rho_new = rho;
    *gamma_new = 1.5;
    return 3;
  }
  *rho_new = a.ok ? a.step : b.step;
  *gamma_new = a.ok ? 1.9 : 1.1;
  return a.ok ? 1 : 2;
}

// merged coefficients of C (Eq. 23): c_prim = sum of rho_i over sets having
// a block of that primitive, times 1/h^2 for the differences
template <class T>
__device__ __host__ inline void make_coeffs(const Prob<T>& P, const double* rho, double* cI, double* cz,
                                            double* cy, double* cx, double* cF) {
  double c[NPRIM] = {0, 0, 0, 0, 0};
  for (int i = 0; i < P.P; ++i)
    for (int b = 0; b < P.set[i].nblk; ++b) c[P.set[i].prim[b]] += rho[i];
  *cI = c[PRIM_I];
  *cz = c[PRIM_Z] * P.g.ihz * P.g.ihz;
  *cy = c[PRIM_Y] * P.g.ihy * P.g.ihy;
  *cx = c[PRIM_X] * P.g.ihx * P.g.ihx;
  *cF = c[PRIM_F];
}

template <class T>
__device__ inline void reset_jobs(const Prob<T>& P, Ctrl& C) {
  for (int jb = 0; jb < C.njobs; ++jb) {
    Job& J = C.job[jb];
    const int i = J.set;
    J.round = 0; J.prefix = 0ull; J.cnt_above = 0; J.sum_above = 0.0; J.cand_n = 0u; J.width = 0ull;
    J.theta = 0.0; J.tau = 0ull; J.keep_eq = 0; J.cnt_eq = 0; J.ties = 0; J.tau_val2 = 0.0;
    J.sigma = C.sigma[i];
    J.k = C.kcard[i];
    J.mode = JM_SEARCH;
    if (J.kind == K_CARD) {
      if (J.k <= 0) J.mode = JM_ZERO;
      else if (J.k >= C.mreal[i]) J.mode = JM_ALL;
    }
  }
}

template <class T>
__device__ void control_body(const Prob<T>& P, Ctrl& C) {
  if (C.stopped) return;
  if (C.numeric_err) { C.stopped = 1; return; }   // set by a kernel (variant mismatch)
  const int k = C.k;
  const int Pn = P.P, p = P.p;
  const bool adapt = is_adapt_it(k, C.opt.adapt_every);
  const bool check = (k % C.opt.check_every) == 0;
  if (k - 1 < C.log_len) C.log_cg[k - 1] = C.cg_count;
  C.cg_total += C.cg_count;
  // NaN guard
  bool bad = !(C.rr == C.rr) || !(C.bb == C.bb);
  for (int i = 0; i < Pn; ++i)
    for (int q = 0; q < NSLOT; ++q) if (!(C.sums[i][q] == C.sums[i][q])) bad = true;
  if (bad) { C.numeric_err = 1; C.stopped = 1; return; }
  if (check) {
    bool feas_ok = true;
    for (int i = 0; i < p; ++i) {
      const int kd = P.set[i].kind;
      const double s2 = C.sums[i][SLOT_S2];
      double fn = C.sums[i][SLOT_FN];
      if (P.set[i].fib || P.set[i].svd) {
        // per-fiber sets: the fiber kernels' sum of per-fiber ||s - P(s)||^2;
        // rank / nuclear sets: k_svdproj's ||s - P(s)||^2
      } else if ((kd == K_L1 || kd == K_CARD) && P.set[i].sjob >= 0) {
        const Job& J = C.job[P.set[i].sjob];
        if (J.mode == JM_INSIDE || J.mode == JM_ALL) fn = 0.0;
        else if (J.mode == JM_ZERO) fn = s2;
        else if (kd == K_CARD) fn += (double)(J.cnt_eq - J.keep_eq) * J.tau_val2;
      } else if (kd == K_L2 || kd == K_ANN) {
        const double n = sqrt(s2);
        double c = n;
        if (n > C.sig_hi[i]) c = C.sig_hi[i];
        else if (n < C.sig_lo[i]) c = C.sig_lo[i];
        fn = (n - c) * (n - c);
      }
      double r;
      if (s2 == 0.0) r = C.zin[i] ? 0.0 : INFINITY;   // reading L19
      else r = sqrt(fn) / sqrt(s2);                          // Eq. 26
      C.r_feas[i] = r;
      if (!(r < C.opt.eps_feas)) feas_ok = false;
      if (k - 1 < C.log_len) C.log_feas[(size_t)(k - 1) * p + i] = r;
    }
    const double xn = sqrt(C.evol[0]);
    double mx = 0.0;
    for (int jj = 0; jj < C.hist_count; ++jj) {
      const int js = (C.hist_head - jj + HIST_S) % HIST_S;
      const double d = sqrt(C.evol[1 + js]);
      if (d > mx) mx = d;
    }
    const double re = xn > 0.0 ? mx / xn : (mx > 0.0 ? INFINITY : 0.0);   // Eq. 27
    C.r_evol = re;
    if (k - 1 < C.log_len) C.log_evol[k - 1] = re;
    if (re < C.opt.eps_evol && feas_ok) {                               // Eq. 28
      C.converged = 1;
      if (!C.opt.fixed_work) {
        C.stopped = 1;
        if (k - 1 < C.log_len)
          for (int i = 0; i < Pn; ++i) {
            C.log_branch[(size_t)(k - 1) * Pn + i] = -1;
            C.log_rho[(size_t)(k - 1) * Pn + i] = C.rho[i];
            C.log_gamma[(size_t)(k - 1) * Pn + i] = C.gamma[i];
          }
        return;
      }
    }
  }
  C.hist_head = (C.hist_head + 1) % HIST_S;
  if (C.hist_count < HIST_S) C.hist_count += 1;
  int br[MAXP];
  for (int i = 0; i < Pn; ++i) br[i] = -1;
  if (adapt) {
    if (C.first_adapt_done) {
      for (int i = 0; i < Pn; ++i) {
        const double* s = C.sums[i];
        const SpecStep a = spectral_step(s[SLOT_HV], s[SLOT_HH], s[SLOT_VHVH], C.opt.eps_corr);
        const SpecStep b = spectral_step(s[SLOT_GV], s[SLOT_GG], s[SLOT_VV], C.opt.eps_corr);
        double rn, gn;
        br[i] = alg2_table(a, b, C.rho[i], &rn, &gn);
        C.rho[i] = rn;
        C.gamma[i] = fmin(fmax(gn, 1.0), C.opt.gamma_max);   // reading L15
      }
      for (int i = 0; i < p; ++i) {                    // reading L16
        const double lo = C.rho[p] / C.opt.rho_ratio_cap, hi = C.rho[p] * C.opt.rho_ratio_cap;
        if (C.rho[i] < lo) C.rho[i] = lo;
        if (C.rho[i] > hi) C.rho[i] = hi;
      }
      make_coeffs(P, C.rho, &C.cI, &C.cz, &C.cy, &C.cx, &C.cF);    // replaces Eq. 24
    }
    C.first_adapt_done = 1;
    C.adapt_calls += 1;
  }
  if (k - 1 < C.log_len)
    for (int i = 0; i < Pn; ++i) {
      C.log_branch[(size_t)(k - 1) * Pn + i] = br[i];
      C.log_rho[(size_t)(k - 1) * Pn + i] = C.rho[i];
      C.log_gamma[(size_t)(k - 1) * Pn + i] = C.gamma[i];
    }
  for (int i = 0; i < Pn; ++i)
    for (int q = 0; q < NSLOT; ++q) C.sums[i][q] = 0.0;
  reset_jobs(P, C);
  C.k = k + 1;
  if (C.k > C.opt.max_iter) C.stopped = 1;
}

// k_control: one thread runs Algorithm 2 / Eq. 26-28 on a shared-memory copy
// of the control block (its ~9 KB moved in and out by the whole CTA), so the
// long chain of dependent reads and writes stays on chip
template <class T>
__global__ void __launch_bounds__(BLOCK) k_control(const __grid_constant__ Prob<T> P) {
  pdl_begin();
  __shared__ Ctrl Cs;
  static_assert(sizeof(Ctrl) % 8 == 0, "Ctrl is copied in 8-byte words");
  constexpr int NW8 = (int)(sizeof(Ctrl) / 8);
  const unsigned long long* g = reinterpret_cast<const unsigned long long*>(P.ctrl);
  unsigned long long* sm = reinterpret_cast<unsigned long long*>(&Cs);
  for (int i = threadIdx.x; i < NW8; i += BLOCK) sm[i] = g[i];
  __syncthreads();
  if (threadIdx.x == 0) control_body<T>(P, Cs);
  __syncthreads();
  unsigned long long* gw = reinterpret_cast<unsigned long long*>(P.ctrl);
  for (int i = threadIdx.x; i < NW8; i += BLOCK) gw[i] = sm[i];
}

// init finaliser (one thread): relative parameters from the norms of A_i m
// (readings L4, L23), cardinality k, select jobs
template <class T>
__device__ inline void fin_init(const Prob<T>& P, Ctrl& C, const double* stage) {
  for (int i = 0; i < P.p; ++i) {
    const double n1 = stage[2 * i], n2 = sqrt(stage[2 * i + 1]);
    const int kd = P.set[i].kind, rel = C.rel[i];
    double sg = C.u_sigma[i], lo = C.u_sig_lo[i], hi = C.u_sig_hi[i];
    if (rel && kd == K_L1) sg *= n1;
    if (rel && kd == K_L2) sg *= n2;
    if (rel && kd == K_ANN) { lo *= n2; hi *= n2; }
    if (kd == K_L2) { lo = 0.0; hi = sg; }
    C.sigma[i] = sg; C.sig_lo[i] = lo; C.sig_hi[i] = hi;
    C.kcard[i] = (rel && kd == K_CARD) ? (long long)floor(C.u_kfrac[i] * (double)C.mreal[i]) : C.u_k[i];
  }
  for (int i = 0; i < MAXP; ++i) { C.ann_scale[i] = 1.0; C.ann_zero[i] = 0; }
  reset_jobs(P, C);
}

// ------------------------------------------------------------ init
// x = m (unless warm), y_i = A_i m, v_i = 0 (reading L13), zero work fields,
// norms of A_i m for relative parameters (readings L4, L23)
template <class T>
__global__ void __launch_bounds__(BLOCK) k_init(const __grid_constant__ Prob<T> P, int init_x, int init_yv) {
  Ctrl& C = *P.ctrl;
  extern __shared__ double acc[];
  __shared__ double sh[NWARP + 1];
  const Geo& g = P.g;
  const int nv = P.P * 2;
  for (int v = threadIdx.x; v < NWARP * nv; v += BLOCK) acc[v] = 0.0;
  __syncthreads();
  const int ntile = (g.N + BLOCK - 1) / BLOCK;
  for (int tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
    const int pt = tile * BLOCK + threadIdx.x;
    const bool valid = pt < g.N;
    Loc L{0, 0, 0, 0};
    if (valid) {
      L = locate(g, pt);
      if (init_x) P.x[pt] = P.m[pt];
      P.hist[0][pt] = P.x[pt];
      // the Alg. 2 snapshots (xs, vh0), the other y / v parity and the
      // global sets' w / s are written before any read, pads included, by
      // the vectorised pass kernels; the scalar kernels and the fiber
      // kernels leave pads alone, so they get zeros (P.init_zero, per set
      // S.fib).  SIP_POISON=1 fills the skipped ones with NaN to prove it.
      if (P.init_zero) { P.xs[0][pt] = (T)0; P.xs[1][pt] = (T)0; }
      else if (P.poison) { P.xs[0][pt] = (T)NAN; P.xs[1][pt] = (T)NAN; }
    }
    for (int i = 0; i < P.P; ++i) {
      const SetD<T>& S = P.set[i];
      double n1 = 0.0, n2 = 0.0;
      for (int bl = 0; bl < S.nblk; ++bl) {
        if (!valid) continue;
        const int64_t off = (int64_t)bl * g.ld + pt;
        const bool pad = is_pad(g, S.prim[bl], L, pt);
        const double am = pad ? 0.0 : prim_fwd(g, P.taps, S.prim[bl], VF<T>{P.m}, pt, L);
        n1 += fabs(am);
        n2 += am * am;
        if (init_yv) { S.y[1][off] = (T)am; S.v[1][off] = (T)0; }
        if (P.init_zero || S.fib || S.svd) {
          S.y[0][off] = (T)0; S.v[0][off] = (T)0; S.vh0[off] = (T)0;
          if (S.w) S.w[off] = (T)0;
          if (S.s) S.s[off] = (T)0;
        } else if (P.poison) {
          S.y[0][off] = (T)NAN; S.v[0][off] = (T)NAN; S.vh0[off] = (T)NAN;
          if (S.w) S.w[off] = (T)NAN;
          if (S.s) S.s[off] = (T)NAN;
        }
      }
      warp_acc(acc, nv, 2 * i, n1);
      warp_acc(acc, nv, 2 * i + 1, n2);
    }
  }
  double* stage = P.partials + (size_t)gridDim.x * nv;
  if (finish_reduction(acc, nv, P.partials, P.counter, stage, sh)) {
    if (P.nranks > 1) publish(P, stage, nv, threadIdx.x, BLOCK);
    else if (threadIdx.x == 0) fin_init<T>(P, C, stage);
  }
}

}  // namespace sip
