// sip_device.cuh -- device-side data structures and helpers of the PARSDMM
// hot path (arXiv 1902.09699) for sm_100a.  Product code: shares nothing with
// oracle/.  Citations P:n = PAPER.md line n; L<n> = DESIGN.md readings.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sip {

constexpr int MAXP = 17;        // p <= 16 sets + the distance block
constexpr int NSLOT = 9;        // per-set reduction slots (see SLOT_*)
constexpr int NEVOL = 6;        // ||x||^2 and ||x - x_hist[j]||^2, j < 5 (Eq. 27)
constexpr int HIST_S = 5;       // s = 5
constexpr int NBUCK = 2048;     // radix digits of 11 bits
constexpr int BLOCK = 256;      // threads per CTA of the streaming kernels
constexpr int NWARP = BLOCK / 32;
constexpr int MAXJOBS = 2 * MAXP;
constexpr int MAXTAPS = 81;     // blur kernel up to 9 x 9
constexpr int GHOST = 2;        // ghost planes on each side of every N-field
constexpr int MAXCG = 16;       // p-vector ring of the deferred x update (n_cg <= MAXCG)

// primitive operators: every set's operator is a stack of 1..3 primitive blocks
enum Prim { PRIM_I = 0, PRIM_Z = 1, PRIM_Y = 2, PRIM_X = 3, PRIM_F = 4, NPRIM = 5 };
// set kinds (Table 1) + the distance block A_{p+1} = I (Eq. 17, 22)
enum Kind { K_BOUNDS = 0, K_L1 = 1, K_L2 = 2, K_ANN = 3, K_CARD = 4, K_DIST = 5, K_RANK = 6, K_NUC = 7 };

// reduction slots per set (fp64)
enum Slot {
  SLOT_W2 = 0,    // ||w||^2                      (l2 / annulus projection)
  SLOT_HV = 1,    // dh . dvh                     (Alg. 2, alpha side)
  SLOT_HH = 2,    // dh . dh
  SLOT_VHVH = 3,  // dvh . dvh
  SLOT_GV = 4,    // dg . dv                      (Alg. 2, beta side)
  SLOT_GG = 5,    // dg . dg
  SLOT_VV = 6,    // dv . dv
  SLOT_FN = 7,    // ||s - P(s)||^2               (Eq. 26 numerator)
  SLOT_S2 = 8     // ||s||^2                      (Eq. 26 denominator)
};

// select-job modes
enum JobMode { JM_OFF = 0, JM_SEARCH = 1, JM_INSIDE = 2, JM_ZERO = 3, JM_DONE = 4, JM_ALL = 5 };

// unsigned 32-bit division by a runtime constant: q = (umulhi(n, m) + n) >> l
struct FastDiv {
  uint32_t d, m, l;
  __host__ void init(uint32_t div) {
    d = div;
    l = 0;
    while ((1ull << l) < div) ++l;
    m = (uint32_t)(((1ull << 32) * ((1ull << l) - div)) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    uint64_t t = (uint64_t)__umulhi(n, m) + n;
    return (uint32_t)(t >> l);
  }
};

struct Geo {
  int ndim;
  int nz, ny, nx;        // local counts (ny = 1 in 2D); nz = slab planes
  int nz_g, z0;          // global nz and the slab's first plane
  int plane, N;          // ny*nx, nz*plane (local points)
  int64_t ld;            // element stride between blocks of a multi-block field
  double ihz, ihy, ihx;  // 1/h (reading L2)
  int kh, kw;            // blur kernel size (0 if none)
  FastDiv dplane, dnx, dny;
  const uint8_t* mask;   // blur observation mask (N, local) or null
};

struct Loc { int iz, iy, ix, gz; };

__device__ __forceinline__ Loc locate(const Geo& g, int pt) {
  Loc L;
  L.iz = (int)g.dplane.div((uint32_t)pt);
  int r = pt - L.iz * g.plane;
  L.iy = (int)g.dnx.div((uint32_t)r);
  L.ix = r - L.iy * g.nx;
  L.gz = L.iz + g.z0;
  return L;
}

// entry (prim, point) is outside the operator's range (reading L3, L21)
__device__ __forceinline__ bool is_pad(const Geo& g, int prim, const Loc& L, int pt) {
  switch (prim) {
    case PRIM_Z: return L.gz >= g.nz_g - 1;
    case PRIM_Y: return L.iy >= g.ny - 1;
    case PRIM_X: return L.ix >= g.nx - 1;
    case PRIM_F: return g.mask[pt] == 0;
    default: return false;
  }
}

template <class T>
struct SetD {
  int kind, nblk, global;
  int prim[3];
  int job, sjob;          // select jobs on w (every iteration) / on s (check)
  int first_real;         // point index of the first entry (annulus at 0, L7)
  int fib, flen;          // per-fiber application (0 whole; 1 x-, 2 z-fibers) and fiber length
  int fpath;              // 1: warp kernel k_fiberw; 0: CTA-per-fiber sort kernel k_fiber
  int svd;                // rank / nuclear-norm set (sip_svd.cuh)
  int dct;                // l1 ball of the grid's orthonormal DCT (kept inside the set)
  T* y[2];                // ping-pong y_i (parity k & 1), nblk blocks of ld
  T* v[2];
  T* vh0;                 // Alg. 2 snapshot v-hat^{k0}
  T* w;                   // w = x-bar - v/rho (global sets)
  T* s;                   // s = A x on check iterations (global l1/card sets)
  const T* lo_vec;        // per-entry bounds (padded layout) or null
  const T* hi_vec;
  double lo, hi;
};

struct Opts {
  int n_cg, eq25, fixed_work, adapt_every, check_every, max_iter;
  double eps_evol, eps_feas, eps_corr, rho_ratio_cap, gamma_max, cg_tol_floor;
};

struct Job {
  int mode, kind, set, on_s, round;
  unsigned long long prefix;     // resolved high digits of the key
  long long cnt_above;           // entries strictly above the prefix range
  double sum_above;              // their sum of |value|
  double sigma;                  // l1 radius
  long long k;                   // cardinality
  double theta;                  // l1 threshold (JM_DONE)
  unsigned long long tau;        // cardinality k-th key (JM_DONE)
  long long keep_eq;             // how many entries == tau to keep
  long long cnt_eq;              // entries == tau
  int ties;                      // index-ordered tie break needed
  double tau_val2;               // tau value squared (feasibility of card)
  unsigned cand_n;               // candidates compacted by round 2 (rounds >= 3 read them)
  unsigned long long width;      // select v2: the key window [prefix, prefix + width) of the next round
};

struct Ctrl {
  // outer iteration state (Algorithm 1)
  int k, stopped, converged, first_adapt_done, adapt_calls, hist_head, hist_count;
  int breakdown, numeric_err, zero_x;
  // CG state (Eq. 25, reading L18)
  int cg_j, cg_active, cg_count, cg_total;
  double bb, rr, rr_prev, alpha, beta, tol;
  double alph[MAXCG];            // alpha_j of this x-update (deferred x += sum alpha_j p_j)
  // merged operator coefficients of C (Eq. 23/24)
  double cI, cz, cy, cx, cF;
  double rho[MAXP], gamma[MAXP];
  // user set parameters (relative ones are fractions, readings L4, L23)
  double u_sigma[MAXP], u_sig_lo[MAXP], u_sig_hi[MAXP], u_kfrac[MAXP];
  long long u_k[MAXP];
  int rel[MAXP], zin[MAXP];      // relative flag; 0 in C_i (reading L19)
  // resolved set parameters
  double sigma[MAXP], sig_lo[MAXP], sig_hi[MAXP];
  long long kcard[MAXP], mreal[MAXP];
  double ann_scale[MAXP];
  int ann_zero[MAXP];
  // reduction results
  double sums[MAXP][NSLOT];
  double evol[NEVOL];
  double r_feas[MAXP], r_evol;
  int P, p;
  Opts opt;
  Job job[MAXJOBS];
  int njobs;
  // log
  int* log_cg; int* log_branch; double* log_rho; double* log_gamma;
  double* log_feas; double* log_evol;
  unsigned long long* log_supp;  // [log_len * p] cardinality support fingerprints (atomic sums)
  int log_len;
};

// ---------------------------------------------------------------- support fingerprint
// A test instrument, not part of the method: the support of a cardinality
// set after iteration k is logged as the wrapping sum of splitmix64(b N_g +
// global point index) over its non-zero entries (b the block, N_g the global
// point count), so per-iteration supports can be compared with the oracle.
__device__ __forceinline__ unsigned long long supp_mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
// warp-uniform call: one atomic per warp
__device__ __forceinline__ void supp_add_warp(const Ctrl& C, int i, unsigned long long h) {
  const int k = C.k;
  if (!C.log_supp || k - 1 >= C.log_len) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(C.log_supp + (size_t)(k - 1) * C.p + i, h);
}

// ---------------------------------------------------------------- keys
// |v| as an order-preserving unsigned key and its significand / exponent
template <class T> struct KeyT;
template <> struct KeyT<float> {
  using U = uint32_t;
  static constexpr int BITS = 31;        // sign bit is always 0
  static constexpr int ROUNDS = 3;       // 11 + 11 + 9 bits
  __device__ static U key(float v) { return __float_as_uint(v) & 0x7fffffffu; }
  __device__ static float val(U k) { return __uint_as_float(k); }
};
template <> struct KeyT<double> {
  using U = unsigned long long;
  static constexpr int BITS = 63;
  static constexpr int ROUNDS = 6;       // 11 x 5 + 8 bits
  __device__ static U key(double v) {
    return (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffull;
  }
  __device__ static double val(U k) { return __longlong_as_double((long long)k); }
};

// digit layout of round r (1-based): the digit holds key bits [lo, hi)
__host__ __device__ inline void digit_bits(int total_bits, int r, int* lo, int* nb) {
  int hi = total_bits - 11 * (r - 1);
  int l = hi - 11;
  if (l < 0) l = 0;
  *lo = l;
  *nb = hi - l;
}

// exact significand split for the bucket sums: value = (s1 * 2^32 + s0) * 2^(e - bias)
template <class T> struct SigT;
template <> struct SigT<float> {
  __device__ static void split(uint32_t key, unsigned long long* s_hi, unsigned long long* s_lo) {
    uint32_t e = key >> 23, m = key & 0x7fffffu;
    *s_hi = 0;
    *s_lo = (e ? (1u << 23) : 0u) | m;
  }
  __device__ static double scale(uint32_t key) {   // 2^(max(e,1) - 150)
    int e = (int)(key >> 23);
    return ldexp(1.0, (e ? e : 1) - 150);
  }
};
template <> struct SigT<double> {
  __device__ static void split(unsigned long long key, unsigned long long* s_hi,
                               unsigned long long* s_lo) {
    unsigned long long e = key >> 52, m = key & 0xfffffffffffffull;
    unsigned long long sig = (e ? (1ull << 52) : 0ull) | m;
    *s_hi = sig >> 32;
    *s_lo = sig & 0xffffffffull;
  }
  __device__ static double scale(unsigned long long key) {  // 2^(max(e,1) - 1075)
    int e = (int)(key >> 52);
    return ldexp(1.0, (e ? e : 1) - 1075);
  }
};

// ---------------------------------------------------------------- launch overlap
// Programmatic dependent launch: the runtime launches the hot kernels with
// cudaLaunchAttributeProgrammaticStreamSerialization, so kernel n+1 may be
// scheduled while kernel n drains (its last-CTA reduction, its tail CTAs).
// Every such kernel starts with pdl_begin(): wait until the previous kernel
// has completed and its memory is visible, then allow the next kernel to
// launch once all of this kernel's CTAs are running.  Without the launch
// attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

// ---------------------------------------------------------------- reductions
// fixed-order block sum (warp shuffle tree, then warps in order): deterministic
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;   // lane 0 holds the sum
}

__device__ inline double block_sum(double v, double* sh /* >= NWARP */) {
  v = warp_sum(v);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NWARP; ++i) t += sh[i];
    sh[0] = t;
  }
  __syncthreads();
  t = sh[0];
  __syncthreads();
  return t;
}

// last-CTA detection (threadfence reduction pattern)
__device__ inline bool last_block(unsigned* counter) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = atomicAdd(counter, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

// last CTA: out[v] = sum over CTAs b of partials[b*nv + v], fixed order.
// Values are spread over the warps (warp w takes v = w, w + NWARP, ...), each
// lane sums a strided subset of the CTAs, then a shuffle tree: no block
// barrier per value, so a wide reduction (pass 1: up to 159 values) costs a
// few L2 round trips instead of one barrier-separated phase per value.
__device__ inline void reduce_partials(const double* partials, int nv, double* out, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nb = (int)gridDim.x;
  if (nv <= 2) {
    // one or two values (the CG scalars): all warps split the CTAs, then the
    // NWARP warp sums are added in order -- one L2 round trip per lane
    __shared__ double ws[2][NWARP];
    const int per = (nb + NWARP - 1) / NWARP;
    const int b0 = w * per, b1 = min(nb, b0 + per);
    for (int v = 0; v < nv; ++v) {
      double a = 0.0;
#pragma unroll 4
      for (int b = b0 + lane; b < b1; b += 32) a += __ldcg(partials + (size_t)b * nv + v);
      a = warp_sum(a);
      if (lane == 0) ws[v][w] = a;
    }
    __syncthreads();
    if (threadIdx.x < nv) {
      double t = 0.0;
      for (int i = 0; i < NWARP; ++i) t += ws[threadIdx.x][i];
      out[threadIdx.x] = t;
    }
    __syncthreads();
    return;
  }
  (void)sh;
  for (int v = w; v < nv; v += NWARP) {
    double a = 0.0;
#pragma unroll 4
    for (int b = lane; b < nb; b += 32) a += __ldcg(partials + (size_t)b * nv + v);
    a = warp_sum(a);
    if (lane == 0) out[v] = a;
  }
  __syncthreads();
}

}  // namespace sip
