// sip_select_small.cuh -- the l1-ball threshold / cardinality k-th key of a
// SMALL job (at most SEL_SMALL_MAX entries, e.g. C1's 64 x 64 TV field) in
// one CTA: the l1 ball by Michelot's fixed point on |w| in shared memory
// (ends on Duchi's active set, reading L5), the cardinality k-th key
// by a bitonic sort of the keys with its tie counts -- one launch instead of the radix rounds, whose
// per-round histogram clears, flushes and serial resolves dominate a
// latency-bound iteration.  One CTA per job; single rank.
#pragma once
#include "sip_fiber.cuh"

namespace sip {

constexpr int SEL_SMALL_MAX = 8192;
__host__ inline size_t selsmall_smem() {
  return (size_t)SEL_SMALL_MAX * (sizeof(unsigned long long) + sizeof(double));
}

__device__ inline void bitonic_keys_desc(unsigned long long* k, int n2) {
  for (int size = 2; size <= n2; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < n2 / 2; t += BLOCK) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool desc = ((lo & size) == 0);
        const unsigned long long a = k[lo], b = k[hi];
        if ((b > a) == desc && a != b) { k[lo] = b; k[hi] = a; }
      }
    }
  __syncthreads();
}

template <class T>
__global__ void __launch_bounds__(BLOCK) k_selsmall(const __grid_constant__ Prob<T> P) {
  using K = KeyT<T>;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  const int jb = blockIdx.x;
  if (jb >= C.njobs) return;
  Job& J = C.job[jb];
  const bool check = (C.k % C.opt.check_every) == 0;
  if (J.mode != JM_SEARCH || (J.on_s && !check)) return;
  extern __shared__ __align__(16) unsigned char ss_raw[];
  unsigned long long* kk = reinterpret_cast<unsigned long long*>(ss_raw);
  double* sm = reinterpret_cast<double*>(kk + SEL_SMALL_MAX);
  __shared__ double sh[NWARP + 1];
  const Geo& g = P.g;
  const SetD<T>& S = P.set[J.set];
  const T* buf = J.on_s ? S.s : S.w;
  const int n = S.nblk * g.N;
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  if (J.kind == K_L1) {
    // l1 ball by Michelot's fixed point on |w| held in shared memory:
    // theta <- (sum_{|w| > theta} |w| - sigma) / #{|w| > theta}, from theta =
    // 0; theta rises monotonically and stops on Duchi's active set (the same
    // exact projection as the sort, reading L5); fixed-order block sums
    for (int q = threadIdx.x; q < n; q += BLOCK) {
      const int bl = q / g.N, pt = q - bl * g.N;
      sm[q] = fabs((double)buf[(int64_t)bl * g.ld + pt]);
    }
    __syncthreads();
    double theta = 0.0, cnt_prev = -1.0;
    double cnt = 0.0, sum = 0.0;
    for (int it = 0; it < 4096; ++it) {
      double c_ = 0.0, s_ = 0.0;
      for (int q = threadIdx.x; q < n; q += BLOCK)
        if (sm[q] > theta) { c_ += 1.0; s_ += sm[q]; }
      cnt = block_sum(c_, sh);
      sum = block_sum(s_, sh);
      if (it == 0 && (sum <= J.sigma || J.sigma <= 0.0)) break;   // inside, or the ball {0}
      if (cnt == cnt_prev) break;                                 // the active set is stable
      cnt_prev = cnt;
      theta = (sum - J.sigma) / cnt;
    }
    if (threadIdx.x == 0) {
      if (sum <= J.sigma && cnt_prev < 0.0) J.mode = JM_INSIDE;   // ||w||_1 <= sigma (L5)
      else if (J.sigma <= 0.0) J.mode = JM_ZERO;
      else { J.theta = theta; J.mode = JM_DONE; }
    }
    return;
  }
  // cardinality: the keys sorted in shared memory, the k-th and its ties
  for (int q = threadIdx.x; q < n2; q += BLOCK) {
    unsigned long long key = 0ull;
    if (q < n) {
      const int bl = q / g.N, pt = q - bl * g.N;
      key = (unsigned long long)K::key(buf[(int64_t)bl * g.ld + pt]);   // pads hold 0
    }
    kk[q] = key;
  }
  bitonic_keys_desc(kk, n2);
  {
    const long long k = J.k;                     // 1 <= k < mreal (reset_jobs handles the rest)
    const unsigned long long tau = kk[k - 1];
    double ab = 0.0, eq = 0.0;
    for (int q = threadIdx.x; q < n2; q += BLOCK) {
      ab += kk[q] > tau ? 1.0 : 0.0;
      eq += kk[q] == tau ? 1.0 : 0.0;
    }
    ab = block_sum(ab, sh);
    eq = block_sum(eq, sh);
    if (threadIdx.x == 0) {
      J.tau = tau;
      J.cnt_above = (long long)ab;
      J.cnt_eq = (long long)eq;
      J.keep_eq = J.k - J.cnt_above;
      J.ties = (J.keep_eq < J.cnt_eq) ? 1 : 0;
      const double tv = (double)K::val((typename K::U)tau);
      J.tau_val2 = tv * tv;
      J.mode = tau == 0ull ? JM_ALL : JM_DONE;
    }
  }
}

}  // namespace sip
