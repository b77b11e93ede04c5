// sip_mich.cuh -- the l1-ball threshold by Michelot's fixed point, warm
// started, in one persistent kernel (sm_100a).
//
// Projection onto {||w||_1 <= sigma} is soft thresholding at the theta of
// Duchi et al. (reading L5).  For any theta <= theta*,
//   f(theta) = (sum_{|w| > theta} |w| - sigma) / #{|w| > theta}
// satisfies theta <= f(theta) <= theta*, and f(theta) = theta exactly when
// the active set {|w| > theta} is the one of theta* (Michelot 1986; it is a
// Newton step on g(t) = sum max(|w| - t, 0) - sigma).  So the iteration
// theta <- f(theta) started anywhere below theta* climbs monotonically to
// the exact threshold and stops when the active count repeats: the same
// active set and the same formula as the sorted algorithm, up to the order
// of the fp64 sum.
//
// Each pass is one streaming read of w with a count and an fp64 sum per
// thread, a fixed-order block sum, and a grid barrier after which every CTA
// reduces the per-CTA partials in the same order (so all CTAs hold the same
// theta).  The kernel is persistent (one wave, every CTA resident) and loops
// on the device until the count repeats.  The start is the job's threshold
// of the previous outer iteration (PARSDMM moves it little), lowered by
// 1e-6 relative; pass 1 also forms ||w||_1 and #{|w| > 0}, so a start above
// theta* (g(start) < sigma) restarts from theta = 0 in the same pass.
// Typical: 2-4 passes warm, ~7 cold, against 3 radix rounds whose
// histograms are shared-atomic bound.  A job still open after MICH_MAX
// passes stays in JM_SEARCH and the radix rounds (k_selectf) finish it.
#pragma once
#include "sip_pass.cuh"

namespace sip {

constexpr int MICH_MAX = 24;
constexpr int MICH_U = 8;   // chunks in flight per thread

template <class T> __device__ __forceinline__ T round_down(double v);
template <> __device__ __forceinline__ float round_down<float>(double v) { return __double2float_rd(v); }
template <> __device__ __forceinline__ double round_down<double>(double v) { return v; }

// grid barrier over co-resident CTAs (bar[0] arrivals, bar[1] generation)
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g0 = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

template <class T>
__global__ void __launch_bounds__(BLOCK) k_mich(const __grid_constant__ Prob<T> P) {
  // no launch_dependents: the next kernel must not take SM space while this
  // grid's CTAs wait for each other at the barriers
  asm volatile("griddepcontrol.wait;" ::: "memory");
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (P.dbg && blockIdx.x == 0 && threadIdx.x == 0)
    printf("k_mich enter k=%d stopped=%d njobs=%d grid=%d\n", C.k, C.stopped, C.njobs, (int)gridDim.x);
  if (C.stopped) return;
  __shared__ double sh[NWARP + 1];
  __shared__ double red[4];
  const bool check = (C.k % C.opt.check_every) == 0;
  const int nch = P.g.N / W;
  const int nb = (int)gridDim.x;
  for (int jb = 0; jb < C.njobs; ++jb) {
    Job& J = C.job[jb];
    if (J.kind != K_L1 || J.mode != JM_SEARCH || J.round != 0 || (J.on_s && !check)) continue;
    const SetD<T>& S = P.set[J.set];
    const T* buf = J.on_s ? S.s : S.w;
    const int tot = S.nblk * nch;
    const double sigma = J.sigma;
    const double th0 = J.theta_w > 0.0 ? J.theta_w * (1.0 - 1e-6) : 0.0;
    double th = th0, cprev = -1.0;
    int pass = 0;
    bool done = false;
    int mode = JM_SEARCH;
    for (; pass < MICH_MAX && !done; ++pass) {
      const bool first = pass == 0;
      // |w| > th in the field's precision: th rounded down to T is the same
      // test for every T-valued |w| (th itself is fp64)
      const T tt = round_down<T>(th);
      long long c = 0, c0 = 0;
      double s = 0.0, s0 = 0.0;
      for (int q0 = blockIdx.x * BLOCK + threadIdx.x; q0 < tot; q0 += nb * BLOCK * MICH_U) {
        T v[MICH_U][W];
#pragma unroll
        for (int u = 0; u < MICH_U; ++u) {   // all loads first (memory-level parallelism)
          const int q = q0 + u * nb * BLOCK;
          const int qq = q < tot ? q : tot - 1;
          const int bl = (qq >= nch) + (qq >= 2 * nch);   // nblk <= 3
          VT<T>::ldT(buf + (int64_t)bl * P.g.ld + (int64_t)(qq - bl * nch) * W, v[u]);
        }
#pragma unroll
        for (int u = 0; u < MICH_U; ++u) {
          if (q0 + u * nb * BLOCK >= tot) continue;
          T cs = 0, cs0 = 0;   // chunk sums in T: W terms, then one fp64 add
#pragma unroll
          for (int e = 0; e < W; ++e) {
            const T a = v[u][e] < (T)0 ? -v[u][e] : v[u][e];
            const bool act = a > tt;
            c += act ? 1 : 0;
            cs += act ? a : (T)0;
            if (first) { c0 += a > (T)0 ? 1 : 0; cs0 += a; }
          }
          s += (double)cs;
          if (first) s0 += (double)cs0;
        }
      }
      const double bc = block_sum((double)c, sh), bs = block_sum(s, sh);
      double bc0 = 0.0, bs0 = 0.0;
      if (first) { bc0 = block_sum((double)c0, sh); bs0 = block_sum(s0, sh); }
      double* part = P.partials + (size_t)(pass & 1) * nb * 4;   // double-buffered by pass parity
      if (threadIdx.x == 0) {
        double* pp = part + (size_t)blockIdx.x * 4;
        pp[0] = bc; pp[1] = bs; pp[2] = bc0; pp[3] = bs0;
      }
      grid_barrier(P.gbar);
      // every CTA: the totals in the same fixed order
      if (threadIdx.x < 32) {
        double a[4] = {0, 0, 0, 0};
        for (int b = threadIdx.x; b < nb; b += 32)
#pragma unroll
          for (int u = 0; u < 4; ++u) a[u] += __ldcg(part + (size_t)b * 4 + u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          double t = a[u];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
          if (threadIdx.x == 0) red[u] = t;
        }
      }
      __syncthreads();
      double Ct = red[0], St = red[1];
      if (first) {
        if (red[3] <= sigma) { mode = JM_INSIDE; done = true; }       // ||w||_1 <= sigma (L5)
        else if (sigma <= 0.0) { mode = JM_ZERO; done = true; }       // the ball is {0}
        else if (!(St - th * Ct >= sigma)) { Ct = red[2]; St = red[3]; }   // start above theta*: from 0
      } else if (Ct == cprev) {
        done = true;   // the active set repeated: th is the fixed point
        mode = JM_DONE;
      }
      if (!done) {
        cprev = Ct;
        th = (St - sigma) / Ct;
      }
      __syncthreads();   // red[] is rewritten by the next pass
    }
    grid_barrier(P.gbar);   // the last partials are read before the next job writes
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      J.mich_passes = (unsigned)pass;
      if (P.dbg) printf("k_mich k=%d job=%d on_s=%d passes=%d mode=%d theta=%.9g start=%.9g\n", C.k, jb, J.on_s, pass,
                        done ? mode : -1, th, th0);
      if (done) {
        J.mode = mode;
        if (mode == JM_DONE) { J.theta = th; J.theta_w = th; }
      }
    }
  }
}

}  // namespace sip
