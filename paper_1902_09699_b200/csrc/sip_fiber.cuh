// sip_fiber.cuh -- per-fiber projections (NEXT-1; "the projection
// onto a simple set is now applied to each row/column independently").
//
// A fiber set's operator output field (single block, grid-shaped, pads 0) is
// split into x-fibers (rows: fixed z, y) or z-fibers (columns: fixed y, x);
// every fiber is projected on its own: cardinality keeps its k largest |w|
// (ties to the lowest index, reading L6), the l1 ball soft-thresholds it at
// the Duchi threshold of its sorted magnitudes (reading L5).  One CTA per
// fiber: the fiber's keys are sorted in shared memory by a bitonic network
// (<= 4096 entries), so the selection is exact and local -- no global
// histogram.  The kernel also forms Algorithm 2's beta-side products and,
// on check iterations, the Eq. 26 numerator ||s - P(s)||^2 of these sets.
#pragma once
#include "sip_pass.cuh"

namespace sip {

constexpr int FIB_MAX = 4096;

// location of entry t of fiber f in the padded field; fibers that are pads
// (D_z x-fibers in the last global plane, D_y x-fibers in the last row,
// D_x z-fibers in the last column) are skipped by the caller
__device__ __forceinline__ int64_t fib_pt(const Geo& g, int mode, int f, int t) {
  if (mode == 1) return (int64_t)f * g.nx + t;                       // f = iz * ny + iy
  const int iy = f / g.nx, ix = f - iy * g.nx;                       // f = iy * nx + ix
  return ((int64_t)t * g.ny + iy) * g.nx + ix;
}
__device__ __forceinline__ bool fib_is_pad(const Geo& g, int mode, int prim, int f) {
  if (mode == 1) {
    const int iz = f / g.ny, iy = f - iz * g.ny;
    return (prim == PRIM_Z && iz + g.z0 >= g.nz_g - 1) || (prim == PRIM_Y && iy >= g.ny - 1);
  }
  const int iy = f / g.nx, ix = f - iy * g.nx;
  return (prim == PRIM_X && ix >= g.nx - 1) || (prim == PRIM_Y && iy >= g.ny - 1);
}

// bitonic sort of n2 (power of 2) (key, index) pairs in shared memory into
// descending key order, equal keys by ascending index (reading L6)
__device__ inline void bitonic_desc(unsigned long long* k, short* ix, int n2) {
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < n2 / 2; t += BLOCK) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool desc = ((lo & size) == 0);
        const unsigned long long a = k[lo], b = k[hi];
        const short ia = ix[lo], ib = ix[hi];
        const bool b_first = b > a || (b == a && ib < ia);   // b ranks before a
        if (b_first == desc) { k[lo] = b; k[hi] = a; ix[lo] = ib; ix[hi] = ia; }
      }
    }
  }
  __syncthreads();
}

// inclusive prefix sums of u[0..L) in place (fp64): per-thread contiguous
// runs, then an exclusive scan of the run totals across the CTA
__device__ inline void block_prefix(double* u, int L, double* sh /* >= NWARP */) {
  const int per = (L + BLOCK - 1) / BLOCK;
  const int b = threadIdx.x * per, e = min(L, b + per);
  double run = 0.0;
  for (int t = b; t < e; ++t) run += u[t];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double inc = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  __syncthreads();
  if (lane == 31) sh[w] = inc;
  __syncthreads();
  double off = inc - run;
  for (int q = 0; q < w; ++q) off += sh[q];
  for (int t = b; t < e; ++t) { off += u[t]; u[t] = off; }
  __syncthreads();
}

// projection of one fiber held in v[0..L) (storage precision) into y[0..L);
// keys / ix / sums are scratch.  Exact: cardinality by sorting (|w|, index)
// -- |w| in the field's precision (reading L27) -- and the l1 ball by
// Duchi's sorted prefix sums in fp64 (reading L5).
template <class T>
__device__ void fib_project(int kind, int L, const T* v, T* y, long long k, double sigma, double lo, double hi,
                            unsigned long long* keys, short* ix, double* sums, double* sh) {
  using K = KeyT<T>;
  if (kind == K_L2 || kind == K_ANN) {   // radial scaling into [lo, hi] (Table 1; L2: lo = 0; L7 at 0)
    double a = 0.0;
    for (int t = threadIdx.x; t < L; t += BLOCK) a += (double)v[t] * (double)v[t];
    const double n = sqrt(block_sum(a, sh));
    double f = 1.0;
    if (n > hi) f = hi / n;
    else if (n < lo && n > 0.0) f = lo / n;
    for (int t = threadIdx.x; t < L; t += BLOCK)
      y[t] = n == 0.0 ? ((t == 0 && lo > 0.0) ? (T)lo : (T)0) : (T)((double)v[t] * f);
    __syncthreads();
    return;
  }
  int n2 = 1;
  while (n2 < L) n2 <<= 1;
  if (kind == K_CARD && k >= L) {
    for (int t = threadIdx.x; t < L; t += BLOCK) y[t] = v[t];
    __syncthreads();
    return;
  }
  // the bit pattern of |w| orders magnitudes; padding sorts last (key 0, index >= L)
  for (int t = threadIdx.x; t < n2; t += BLOCK) {
    keys[t] = t < L ? (unsigned long long)K::key(v[t]) : 0ull;
    ix[t] = (short)t;
  }
  bitonic_desc(keys, ix, n2);
  if (kind == K_CARD) {   // keep the first k in (|w| desc, index asc) order
    for (int t = threadIdx.x; t < L; t += BLOCK) y[t] = (T)0;
    __syncthreads();
    for (int j = threadIdx.x; j < L && j < k; j += BLOCK) y[ix[j]] = v[ix[j]];
    __syncthreads();
    return;
  }
  // l1 ball: u = sorted |w|, S_j = u_1 + ... + u_j
  for (int t = threadIdx.x; t < L; t += BLOCK) sums[t] = (double)K::val((typename K::U)keys[t]);
  __syncthreads();
  block_prefix(sums, L, sh);
  __shared__ int s_rho;
  __shared__ double s_theta;
  if (threadIdx.x == 0) s_rho = 0;
  __syncthreads();
  const double tot = L > 0 ? sums[L - 1] : 0.0;
  const bool inside = tot <= sigma;
  if (!inside && sigma > 0.0) {   // largest j with u_j - (S_j - sigma) / j > 0 (Duchi)
    for (int t = threadIdx.x; t < L; t += BLOCK) {
      const double u = (double)K::val((typename K::U)keys[t]);
      if (u - (sums[t] - sigma) / (double)(t + 1) > 0.0) atomicMax(&s_rho, t + 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) s_theta = s_rho > 0 ? (sums[s_rho - 1] - sigma) / (double)s_rho : 0.0;
  __syncthreads();
  const double th = s_theta;
  for (int t = threadIdx.x; t < L; t += BLOCK) {
    const T w = v[t];
    if (inside) { y[t] = w; continue; }
    if (sigma <= 0.0) { y[t] = (T)0; continue; }
    const double a = fabs((double)w) - th;
    y[t] = a > 0.0 ? (T)(w > (T)0 ? a : -a) : (T)0;
  }
  __syncthreads();
}

// k_fiber: y = P(w) per fiber, v = rho (y - w) (L26), Alg. 2 beta-side sums,
// Eq. 26 numerator on s (check iterations); sums land in C.sums like pass 2's
template <class T>
__global__ void __launch_bounds__(BLOCK) k_fiber(const __grid_constant__ Prob<T> P) {
  pdl_begin();
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  extern __shared__ __align__(16) unsigned char fsm[];
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(fsm);        // [FIB_MAX]
  double* sums = reinterpret_cast<double*>(keys + FIB_MAX);                      // [FIB_MAX]
  T* vin = reinterpret_cast<T*>(sums + FIB_MAX);                                 // [FIB_MAX]
  T* vout = vin + FIB_MAX;                                                       // [FIB_MAX]
  short* ix = reinterpret_cast<short*>(vout + FIB_MAX);                          // [FIB_MAX]
  __shared__ double sh[NWARP + 1];
  __shared__ double out[4 * MAXP];
  const Geo& g = P.g;
  const IterFlags f = iter_flags<2, 2>(C);
  const int par = C.k & 1;
  double acc[4] = {0, 0, 0, 0};
  __shared__ double accs[4 * MAXP];
  for (int v = threadIdx.x; v < 4 * MAXP; v += BLOCK) accs[v] = 0.0;
  __syncthreads();
  for (int i = 0; i < P.P; ++i) {
    const SetD<T>& S = P.set[i];
    if (!S.fib || S.fpath) continue;
    const int prim = S.prim[0];
    const int nfib = S.fib == 1 ? g.nz * g.ny : g.ny * g.nx;
    const int L = S.flen;
    const T rho = (T)C.rho[i];
    const long long kk = C.kcard[i];
    const double sg = C.sigma[i], slo = C.sig_lo[i], shi = C.sig_hi[i];
    T* yw = S.y[par ^ 1];
    T* vw = S.v[par ^ 1];
    acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
    for (int fb = blockIdx.x; fb < nfib; fb += gridDim.x) {
      if (fib_is_pad(g, S.fib, prim, fb)) continue;
      for (int t = threadIdx.x; t < L; t += BLOCK) vin[t] = S.w[fib_pt(g, S.fib, fb, t)];
      __syncthreads();
      fib_project<T>(S.kind, L, vin, vout, kk, sg, slo, shi, keys, ix, sums, sh);
      for (int t = threadIdx.x; t < L; t += BLOCK) {
        const int64_t pt = fib_pt(g, S.fib, fb, t);
        const T y = vout[t];
        const T vt = rho * (y - vin[t]);                 // Eq. 21 as rho (y - w), L26
        if (f.dots) {
          const T dg = yw[pt] - y, dv = vt - vw[pt];
          acc[0] += (double)(dg * dv); acc[1] += (double)(dg * dg); acc[2] += (double)(dv * dv);
        }
        yw[pt] = y;
        vw[pt] = vt;
      }
      __syncthreads();
      if (f.check && S.s) {   // Eq. 26 numerator: the per-fiber projection of s
        for (int t = threadIdx.x; t < L; t += BLOCK) vin[t] = S.s[fib_pt(g, S.fib, fb, t)];
        __syncthreads();
        fib_project<T>(S.kind, L, vin, vout, kk, sg, slo, shi, keys, ix, sums, sh);
        for (int t = threadIdx.x; t < L; t += BLOCK) {
          const double d = (double)vin[t] - (double)vout[t];
          acc[3] += d * d;
        }
        __syncthreads();
      }
    }
    for (int q = 0; q < 4; ++q) {
      const double a = block_sum(acc[q], sh);
      if (threadIdx.x == 0) accs[4 * i + q] = a;
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < 4 * P.P; v += BLOCK) P.partials[(size_t)blockIdx.x * 4 * P.P + v] = accs[v];
  if (last_block(P.counter)) {
    reduce_partials(P.partials, 4 * P.P, out, sh);
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      for (int i = 0; i < P.P; ++i) {
        if (!P.set[i].fib || P.set[i].fpath) continue;
        if (P.nranks > 1) {   // z slabs: rank-local, summed with pass 2's values
          for (int q = 0; q < 4; ++q) P.fibv[4 * i + q] = out[4 * i + q];
          continue;
        }
        C.sums[i][SLOT_GV] = out[4 * i + 0];
        C.sums[i][SLOT_GG] = out[4 * i + 1];
        C.sums[i][SLOT_VV] = out[4 * i + 2];
        C.sums[i][SLOT_FN] = out[4 * i + 3];
      }
    }
  }
}

__host__ inline size_t fiber_smem(int dsize) { return (size_t)FIB_MAX * (8 + 8 + 2 * dsize + 2); }

// ---------------------------------------------------------------------------
// k_fiberw: one warp per fiber, the fiber in registers (E entries per lane,
// entry t = e * 32 + lane, fibers of <= 32 * FW_E entries).  No sort; every
// step is a warp-wide count / sum:
//  - cardinality: a bitwise search over the |w| key space (<= 31 steps fp32,
//    63 fp64) for tau = the k-th largest key, the largest key with
//    #{key >= tau} >= k.  A candidate with #{key >= cand} == k exactly ends
//    the search ({key >= cand} is the top k, nothing to break); otherwise
//    keep key > tau and the first k - #{key > tau} entries equal to tau in
//    index order (ballot prefix, reading L6);
//  - l1 ball: Michelot's fixed point theta = (sum_{|w| > theta} |w| - sigma)
//    / #{|w| > theta}, started from theta = (||w||_1 - sigma) / L.  theta
//    grows and the active set shrinks monotonically, and the fixed point is
//    the theta of Duchi's sorted algorithm (reading L5): the same active set
//    (rho entries) and the same sum; it usually settles in a few steps.
// x-fibers are contiguous rows: each warp reads its row straight from HBM;
// z-fibers (stride ny*nx) go through a shared tile of FW_TC adjacent columns
// x L planes so every HBM access is a coalesced row segment.
constexpr int FW_E = 16;
constexpr int FW_TS = 4;                 // z tiles: 2^FW_TS adjacent columns (64-byte fp32 row segments)
constexpr int FW_TC = 1 << FW_TS;
constexpr int FW_TP = FW_TC + 1;         // tile pitch (+1: conflict-free column reads)

__device__ __forceinline__ double fw_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int fw_cnt(int v) { return __reduce_add_sync(0xffffffffu, v); }

template <class T, int E>
__device__ __forceinline__ void fw_project_e(int kind, const T* w, T* y, long long k, double sigma, double lo,
                                             double hi, int L, int lane) {
  using K = KeyT<T>;
  using U = typename K::U;
  if (kind == K_L2 || kind == K_ANN) {   // radial scaling into [lo, hi] (Table 1; L2: lo = 0; L7 at 0)
    double a = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) a += (double)w[e] * (double)w[e];
    const double n = sqrt(fw_sum(a));
    double f = 1.0;
    if (n > hi) f = hi / n;
    else if (n < lo && n > 0.0) f = lo / n;
#pragma unroll
    for (int e = 0; e < E; ++e)
      y[e] = n == 0.0 ? ((e == 0 && lane == 0 && lo > 0.0) ? (T)lo : (T)0) : (T)((double)w[e] * f);
    return;
  }
  if (kind == K_CARD) {
    if (k >= L) {
#pragma unroll
      for (int e = 0; e < E; ++e) y[e] = w[e];
      return;
    }
    if (k <= 0) {
#pragma unroll
      for (int e = 0; e < E; ++e) y[e] = (T)0;
      return;
    }
    U key[E];   // |w| bit patterns, formed once
#pragma unroll
    for (int e = 0; e < E; ++e) key[e] = K::key(w[e]);
    U tau = 0;   // entries past L are 0: key 0 never reaches a candidate >= 1
    bool exact = false;
    for (int b = K::BITS - 1; b >= 0; --b) {
      const U cand = tau | ((U)1 << b);
      int c = 0;
#pragma unroll
      for (int e = 0; e < E; ++e) c += key[e] >= cand ? 1 : 0;
      c = fw_cnt(c);
      if (c >= k) {
        tau = cand;
        if (c == k) { exact = true; break; }   // {key >= tau} is the top k: no tie to break
      }
    }
    if (exact) {
#pragma unroll
      for (int e = 0; e < E; ++e) y[e] = key[e] >= tau ? w[e] : (T)0;
      return;
    }
    if (tau == 0) {   // fewer than k nonzeros: every nonzero kept, the rest is 0 = w
#pragma unroll
      for (int e = 0; e < E; ++e) y[e] = w[e];
      return;
    }
    int gt = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) gt += key[e] > tau ? 1 : 0;
    const long long need = k - fw_cnt(gt);
    const unsigned lt = (1u << lane) - 1u;
    int run = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const unsigned tie = __ballot_sync(0xffffffffu, key[e] == tau);
      const bool keep = key[e] > tau || (key[e] == tau && run + __popc(tie & lt) < need);
      run += __popc(tie);
      y[e] = keep ? w[e] : (T)0;
    }
    return;
  }
  double a[E];   // |w| in fp64, formed once
  double a1 = 0.0;
#pragma unroll
  for (int e = 0; e < E; ++e) { a[e] = fabs((double)w[e]); a1 += a[e]; }
  const double tot = fw_sum(a1);
  if (tot <= sigma) {
#pragma unroll
    for (int e = 0; e < E; ++e) y[e] = w[e];
    return;
  }
  if (sigma <= 0.0) {
#pragma unroll
    for (int e = 0; e < E; ++e) y[e] = (T)0;
    return;
  }
  // Michelot's fixed point: theta = (sum of the active |w| - sigma) / #active
  // over the active set {|w| > theta}; theta only grows, the active set only
  // shrinks, and the fixed point is Duchi's theta (same rho, same sum).
  double th = (tot - sigma) / (double)L;
  int na = L;
  for (;;) {
    int c = 0;
    double s1 = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if (a[e] > th) { ++c; s1 += a[e]; }
    c = fw_cnt(c);
    if (c == na) break;   // warp-uniform
    s1 = fw_sum(s1);
    na = c;
    th = (s1 - sigma) / (double)na;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const double d = a[e] - th;
    y[e] = d > 0.0 ? (T)(w[e] > (T)0 ? d : -d) : (T)0;
  }
}

// shared bytes of the z-fiber tiles (w and y, L x FW_TP each)
__host__ __device__ inline size_t fiberw_smem(int L, int dsize) { return (size_t)2 * L * FW_TP * dsize; }
// entries per lane for a fiber length (the kernel instantiation)
__host__ __device__ inline int fiberw_e(int L) { return L <= 128 ? 4 : L <= 256 ? 8 : 16; }

// one launch per fiber set i; E = fiberw_e(flen).  The previous y / v (Alg. 2
// products) are loaded before the threshold search so their latency hides
// behind it; z tiles move through shared memory in batches of FW_U rows.
constexpr int FW_U = 16;

template <class T, int E>
__global__ void __launch_bounds__(BLOCK, E <= 8 ? 3 : 1) k_fiberw(const __grid_constant__ Prob<T> P, int i) {
  pdl_begin();
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  extern __shared__ __align__(16) unsigned char fsm[];
  __shared__ double sh[NWARP + 1];
  __shared__ double out[4];
  const Geo& g = P.g;
  const IterFlags f = iter_flags<2, 2>(C);
  const int par = C.k & 1;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const SetD<T>& S = P.set[i];
  const int prim = S.prim[0];
  const int L = S.flen;
  const T rho = (T)C.rho[i];
  const long long kk = C.kcard[i];
  const double sg = C.sigma[i], slo = C.sig_lo[i], shi = C.sig_hi[i];
  T* yw = S.y[par ^ 1];
  T* vw = S.v[par ^ 1];
  const bool chk = f.check && S.s;
  double acc[4] = {0, 0, 0, 0};
  T w[E], y[E];
  if (S.fib == 1) {   // x-fibers: a warp per row, straight from HBM
    const int nf = g.nz * g.ny;
    for (int fb = blockIdx.x * NWARP + wid; fb < nf; fb += gridDim.x * NWARP) {
      if (fib_is_pad(g, 1, prim, fb)) continue;
      const int64_t base = (int64_t)fb * g.nx;
      T y0[E], v0[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int t = e * 32 + lane;
        w[e] = t < L ? S.w[base + t] : (T)0;
        y0[e] = (f.dots && t < L) ? yw[base + t] : (T)0;
        v0[e] = (f.dots && t < L) ? vw[base + t] : (T)0;
      }
      fw_project_e<T, E>(S.kind, w, y, kk, sg, slo, shi, L, lane);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int t = e * 32 + lane;
        if (t >= L) continue;
        const T vt = rho * (y[e] - w[e]);                  // Eq. 21 as rho (y - w), L26
        if (f.dots) {
          const T dg = y0[e] - y[e], dv = vt - v0[e];
          acc[0] += (double)(dg * dv); acc[1] += (double)(dg * dg); acc[2] += (double)(dv * dv);
        }
        yw[base + t] = y[e];
        vw[base + t] = vt;
      }
      if (chk) {   // Eq. 26 numerator of this fiber
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int t = e * 32 + lane;
          w[e] = t < L ? S.s[base + t] : (T)0;
        }
        fw_project_e<T, E>(S.kind, w, y, kk, sg, slo, shi, L, lane);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double d = (double)w[e] - (double)y[e];   // 0 past L (w = y = 0 there)
          acc[3] += d * d;
        }
      }
    }
  } else {   // z-fibers: tiles of FW_TC adjacent columns staged in shared memory
    T* tw = reinterpret_cast<T*>(fsm);
    T* ty = tw + (size_t)L * FW_TP;
    const int ntx = (g.nx + FW_TC - 1) / FW_TC;
    const int ntile = g.ny * ntx;
    const int64_t pl = (int64_t)g.plane;
    const int nq = L * FW_TC;
    for (int tl = blockIdx.x; tl < ntile; tl += gridDim.x) {
      const int iy = tl / ntx, ix0 = (tl - iy * ntx) * FW_TC;
      const int64_t b0 = (int64_t)iy * g.nx + ix0;
      const int c_ = threadIdx.x & (FW_TC - 1);
      const bool colok = ix0 + c_ < g.nx && !fib_is_pad(g, 2, prim, iy * g.nx + ix0 + c_);
      for (int ph = 0; ph < (chk ? 2 : 1); ++ph) {
        const T* src = ph == 0 ? S.w : S.s;
        for (int q0 = threadIdx.x; q0 < nq; q0 += BLOCK * FW_U) {   // batched coalesced loads
          T r[FW_U];
#pragma unroll
          for (int u = 0; u < FW_U; ++u) {
            const int q = q0 + u * BLOCK;
            r[u] = (q < nq && ix0 + c_ < g.nx) ? src[(q >> FW_TS) * pl + b0 + c_] : (T)0;
          }
#pragma unroll
          for (int u = 0; u < FW_U; ++u) {
            const int q = q0 + u * BLOCK;
            if (q < nq) tw[(q >> FW_TS) * FW_TP + c_] = r[u];
          }
        }
        __syncthreads();
        for (int c = wid; c < FW_TC; c += NWARP) {
          const int ix = ix0 + c;
          if (ix >= g.nx || fib_is_pad(g, 2, prim, iy * g.nx + ix)) continue;   // warp-uniform
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int t = e * 32 + lane;
            w[e] = t < L ? tw[t * FW_TP + c] : (T)0;
          }
          fw_project_e<T, E>(S.kind, w, y, kk, sg, slo, shi, L, lane);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const int t = e * 32 + lane;
            if (ph == 0) {
              if (t < L) ty[t * FW_TP + c] = y[e];
            } else {
              const double d = (double)w[e] - (double)y[e];
              acc[3] += d * d;
            }
          }
        }
        __syncthreads();
        if (ph == 0) {   // y, v = rho (y - w) and the Alg. 2 sums, coalesced
          for (int q0 = threadIdx.x; q0 < nq; q0 += BLOCK * FW_U) {
            T a0[FW_U], b0v[FW_U];
#pragma unroll
            for (int u = 0; u < FW_U; ++u) {
              const int q = q0 + u * BLOCK;
              const bool ok = q < nq && colok && f.dots;
              a0[u] = ok ? yw[(q >> FW_TS) * pl + b0 + c_] : (T)0;
              b0v[u] = ok ? vw[(q >> FW_TS) * pl + b0 + c_] : (T)0;
            }
#pragma unroll
            for (int u = 0; u < FW_U; ++u) {
              const int q = q0 + u * BLOCK;
              if (q >= nq || !colok) continue;
              const int t = q >> FW_TS;
              const int64_t pt = t * pl + b0 + c_;
              const T wt = tw[t * FW_TP + c_], yt = ty[t * FW_TP + c_];
              const T vt = rho * (yt - wt);
              if (f.dots) {
                const T dg = a0[u] - yt, dv = vt - b0v[u];
                acc[0] += (double)(dg * dv); acc[1] += (double)(dg * dg); acc[2] += (double)(dv * dv);
              }
              yw[pt] = yt;
              vw[pt] = vt;
            }
          }
          __syncthreads();
        }
      }
    }
  }
  double part[4];
  for (int q = 0; q < 4; ++q) part[q] = block_sum(acc[q], sh);
  if (threadIdx.x == 0)
    for (int q = 0; q < 4; ++q) P.partials[(size_t)blockIdx.x * 4 + q] = part[q];
  if (last_block(P.counter)) {
    reduce_partials(P.partials, 4, out, sh);
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      if (P.nranks > 1) {   // z slabs: rank-local, summed with pass 2's values
        for (int q = 0; q < 4; ++q) P.fibv[4 * i + q] = out[q];
      } else {
        C.sums[i][SLOT_GV] = out[0];
        C.sums[i][SLOT_GG] = out[1];
        C.sums[i][SLOT_VV] = out[2];
        C.sums[i][SLOT_FN] = out[3];
      }
    }
  }
}

// the warp kernel instantiation for a fiber length
template <class T>
struct FiberW {
  using F = void (*)(Prob<T>, int);
  static F of(int L) {
    const int E = fiberw_e(L);
    return E == 4 ? k_fiberw<T, 4> : E == 8 ? k_fiberw<T, 8> : k_fiberw<T, 16>;
  }
};

}  // namespace sip
