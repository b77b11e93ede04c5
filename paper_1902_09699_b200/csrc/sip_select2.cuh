// sip_select2.cuh -- the exact l1-ball threshold and cardinality k-th key for
// single-rank fp32 runs (sm_100a), in one streaming pass of w after pass 1.
//
// What is computed is unchanged (readings L5, L6): the l1 ball's
// theta with sum_j max(|w_j| - theta, 0) = sigma (Duchi's active set), or the
// key of the k-th largest |w| with the index-ordered tie count.  The keys are
// the IEEE bit patterns of |w| (monotone for non-negative floats).
//
//   round A  (inside k_pass1t, while w is written): a COUNT histogram of the
//            top 11 key bits of every radix job -- one shared atomic per
//            entry, no second read of w.
//   k_selB   every CTA turns the counts into a candidate key range [lo, hi)
//            that must contain the answer (cardinality: the bucket of the
//            k-th key; l1: bounds of sum max(|w| - e, 0) at every bucket
//            edge e from the counts alone), then streams w once: entries
//            >= hi are summed into (count, sum) in registers, entries in
//            [lo, hi) are appended to the CTA's candidate region.
//   k_selC   2-3 rounds over the candidates only (L2-resident): exact
//            histograms (counts + 16-bit limb sums) of a window of keys that
//            shrinks 2048-fold per round down to a single key.
//
// Replaces three full-read radix rounds with three shared atomics per entry
// each (k_selectf): one full read, one shared atomic per entry in pass 1,
// and the candidate rounds on a small grid.  Multi-rank and
// fp64 runs keep k_selectf (its finalisers gather across ranks).
#pragma once
#include "sip_flat.cuh"

namespace sip {

constexpr int A_SHIFT = 20;                 // round-A digit: key bits 30..20 (11 bits)

__device__ __forceinline__ unsigned key32(float v) { return __float_as_uint(v) & 0x7fffffffu; }
__device__ __forceinline__ double kval(unsigned key) { return (double)__uint_as_float(key); }

// round A: one count per non-zero entry (zeros never decide: a zero never
// displaces a non-zero of the top k and adds nothing to an l1 sum)
// one shared atomic per non-zero entry (grouping the lanes of a warp by
// bucket with __match_any_sync first was measured slower: pass 1 3.24 vs
// 2.65 ms per C4 step)
// With t (l1 jobs, non-check iterations) also the sum of every entry's key
// bits 19..12 (its 1/256 sub-bucket): the bucket's value sum is then known to
// within count x 2^12 ulps, which pins sum_j max(|w_j| - e, 0) at every bucket
// edge to ~1e-4 of itself, so k_selB's l1 window is one bucket wide, as for
// the cardinality count.
constexpr int T_SHIFT = 12;
template <class T>
__device__ __forceinline__ void hist_a(unsigned* h, const T* v, unsigned* t = nullptr) {
  if constexpr (sizeof(T) == 4) {
    constexpr int W = VT<T>::W;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const unsigned k = key32((float)v[e]);
      if (k) {
        atomicAdd(&h[k >> A_SHIFT], 1u);
        if (t) atomicAdd(&t[k >> A_SHIFT], (k >> T_SHIFT) & 0xffu);
      }
    }
  }
}
template <class G>
__device__ __forceinline__ void hist_a_flush(unsigned* h, G* g) {
  __syncthreads();
  for (int d = threadIdx.x; d < NBUCK; d += BLOCK) {
    const unsigned c = h[d];
    if (c) { atomicAdd(g + d, (G)c); h[d] = 0u; }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- ranges
// The candidate range of a job from the round-A counts c_d (bucket d holds
// the keys [d 2^20, (d+1) 2^20), values in [e_d, e_{d+1})).  Computed
// identically by every CTA of k_selB (no serial tail), fixed reduction order.
struct SelRange {
  int mode;            // JM_SEARCH, or a final JM_ZERO / JM_INSIDE / JM_ALL
  unsigned lo, hi;     // candidates lo <= key < hi (non-zero); key >= hi: above
};

// the exclusive suffix (over the threads after this one) of per-thread values,
// fixed order: a warp-level inclusive suffix by shuffles, then the totals of
// the later warps
template <class V>
__device__ __forceinline__ V suffix_excl(V v, V* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  V inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const V t = __shfl_down_sync(0xffffffffu, inc, o);
    if (lane + o < 32) inc += t;
  }
  if (lane == 0) sh[w] = inc;
  __syncthreads();
  V later = (V)0;
  for (int q = NWARP - 1; q > w; --q) later += sh[q];
  __syncthreads();
  return later + inc - v;
}

// the lower edge value of round-A bucket d; the buckets of the inf / NaN
// keys (d >= 0x7f8: exponent 255) never hold entries and get FLT_MAX, so no
// inf (or 0 x inf) enters the sums
__device__ __forceinline__ double edge_a(int d) {
  return d < 0x7f8 ? kval((unsigned)d << A_SHIFT) : 3.4028234663852886e38;
}

// 2^12 ulps of the keys of round-A bucket d (one exponent per bucket)
__device__ __forceinline__ double tstep_a(int d) {
  const int ex = d >> 3;                        // exponent field (11-bit digit = exponent + 3 mantissa bits)
  return ldexp(1.0, (ex ? ex : 1) - 150 + T_SHIFT);
}

__device__ inline SelRange range_of_job(const Job& J, const unsigned* gcnt, const unsigned long long* gta) {
  __shared__ unsigned long long s_u[NWARP];
  __shared__ double s_d[NWARP];
  __shared__ int s_best[2];
  SelRange R{JM_SEARCH, 0u, 0u};
  constexpr int PER = NBUCK / BLOCK;        // 8 buckets per thread
  const int d0 = threadIdx.x * PER;
  unsigned c[PER];
  unsigned long long ct = 0;
  double et = 0.0, e1t = 0.0;
  double lo_[PER], hi_[PER];   // bounds of the bucket's value sum
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int d = d0 + q;
    c[q] = __ldcg(gcnt + d);
    ct += c[q];
    if (gta && d < 0x7f8) {
      const double ts = tstep_a(d);
      const double tq = (double)__ldcg(gta + d);
      lo_[q] = (double)c[q] * edge_a(d) + tq * ts;
      hi_[q] = lo_[q] + (double)c[q] * ts;
    } else {
      lo_[q] = (double)c[q] * edge_a(d);
      hi_[q] = (double)c[q] * edge_a(d + 1);
    }
    et += lo_[q];
    e1t += hi_[q];
  }
  const unsigned long long c_after = suffix_excl<unsigned long long>(ct, s_u);
  const double e_after = suffix_excl<double>(et, s_d);
  const double e1_after = suffix_excl<double>(e1t, s_d);
  if (threadIdx.x == 0) { s_best[0] = -1; s_best[1] = -1; }
  __syncthreads();
  int best_lo = -1, best_hi = -1;
  unsigned long long C = c_after;
  double E = e_after, E1 = e1_after;
#pragma unroll
  for (int q = PER - 1; q >= 0; --q) {       // C, E, E1 over the buckets >= d
    const int d = d0 + q;
    C += c[q];
    const double e = edge_a(d);
    E += lo_[q];
    E1 += hi_[q];
    if (J.kind == K_CARD) {
      if (C >= (unsigned long long)J.k && best_hi < d) best_hi = d;
    } else {
      // f(e_d) = sum_{|w| >= e_d} (|w| - e_d) lies in [E - e_d C, E1 - e_d C];
      // an absolute margin keeps the bounds safe under fp64 rounding
      const double L = E - e * (double)C - 1e-12 * E;
      const double U = E1 - e * (double)C + 1e-12 * E1;
      if (L > J.sigma && best_lo < d) best_lo = d;
      if (U > J.sigma && best_hi < d) best_hi = d;
    }
  }
  if (best_lo >= 0) atomicMax(&s_best[0], best_lo);
  if (best_hi >= 0) atomicMax(&s_best[1], best_hi);
  __syncthreads();
  const int blo = s_best[0], bhi = s_best[1];
  __syncthreads();
  if (J.kind == K_CARD) {
    if (bhi < 0) { R.mode = JM_ALL; return R; }              // fewer than k non-zeros: keep all
    R.lo = (unsigned)bhi << A_SHIFT;
    R.hi = (unsigned)(bhi + 1) << A_SHIFT;
    return R;
  }
  if (J.sigma <= 0.0) { R.mode = JM_ZERO; return R; }        // the ball is {0} (L5)
  if (bhi < 0) { R.mode = JM_INSIDE; return R; }             // ||w||_1 <= U(0) <= sigma
  R.lo = blo < 0 ? 0u : (unsigned)blo << A_SHIFT;
  R.hi = (unsigned)(bhi + 1) << A_SHIFT;
  return R;
}

__device__ __forceinline__ bool job_live(const Job& J, bool check) {
  return J.mode == JM_SEARCH && J.round == 0 && (!J.on_s || check);
}

// ---------------------------------------------------------------- windows
// window [lo, lo + width) split into <= 2048 buckets of 2^shift keys; every
// bucket lies inside one exponent (lo is a multiple of 2^20, shift <= 20),
// so its limb sums are exact multiples of one power of two
__device__ __forceinline__ int sel_shift(unsigned long long width, int dbits) {
  int b = 0;
  while ((1ull << b) < width) ++b;        // ceil(log2(width))
  return b > dbits ? b - dbits : 0;
}
#ifndef SIP_FB_BITS
#define SIP_FB_BITS 9
#endif
constexpr int FB_BITS = SIP_FB_BITS;      // k_selB's histogram of the candidates: 512 buckets, so a
                                          // one-bucket window (2^20 keys) needs one k_selC round, not two
constexpr int FB_N = 1 << FB_BITS;

// last CTA of k_selC: the bucket d* of the window holding the answer (the
// walk of resolve_round over linear sub-buckets), then either the next,
// 2048x narrower window or -- single-key buckets -- the final theta / tau
__device__ void resolve_window(Ctrl& C, Job& J, const unsigned* hc, const unsigned long long* h0, int dbits) {
  __shared__ long long s_cnt[BLOCK];
  __shared__ double s_sum[BLOCK];
  __shared__ unsigned long long s_su[NWARP];
  __shared__ double s_sd[NWARP];
  __shared__ int s_dstar;
  __shared__ long long s_cab;
  __shared__ double s_sab;
  const unsigned lo = (unsigned)J.prefix;
  const int sh = sel_shift(J.width, dbits);
  const int nbk = (int)((J.width + (1ull << sh) - 1) >> sh);
  const int per = (nbk + BLOCK - 1) / BLOCK;
  const int d0 = threadIdx.x * per;
  auto bsum = [&](int d) {     // exact sum of the bucket's values: limbs x 2^(e - 150)
    const unsigned kb = lo + ((unsigned)d << sh);
    return (double)__ldcg(h0 + d) * SigT<float>::scale(kb);
  };
  long long c_loc = 0;
  double s_loc = 0.0;
  for (int d = d0; d < d0 + per && d < nbk; ++d) { c_loc += __ldcg(hc + d); s_loc += bsum(d); }
  // totals of the threads above (fixed order: warp suffix, later warps)
  s_cnt[threadIdx.x] = (long long)suffix_excl<unsigned long long>((unsigned long long)c_loc, s_su);
  s_sum[threadIdx.x] = suffix_excl<double>(s_loc, s_sd);
  if (threadIdx.x == 0) s_dstar = -1;
  __syncthreads();
  long long c_ge = J.cnt_above + s_cnt[threadIdx.x];
  double s_ge = J.sum_above + s_sum[threadIdx.x];
  int best = -1;
  for (int d = min(d0 + per, nbk) - 1; d >= d0; --d) {
    const unsigned kb = lo + ((unsigned)d << sh);
    c_ge += __ldcg(hc + d);
    s_ge += bsum(d);
    const bool ok = (J.kind == K_L1) ? (s_ge - kval(kb) * (double)c_ge) > J.sigma   // f(e_d) > sigma
                                     : c_ge >= J.k;                                 // C(>= d) >= k
    if (ok && d > best) best = d;
  }
  if (best >= 0) atomicMax(&s_dstar, best);
  __syncthreads();
  const int dstar = s_dstar;
  if (dstar >= d0 && dstar < d0 + per) {   // totals strictly above d*
    long long c = J.cnt_above + s_cnt[threadIdx.x];
    double sm = J.sum_above + s_sum[threadIdx.x];
    for (int d = min(d0 + per, nbk) - 1; d > dstar; --d) { c += __ldcg(hc + d); sm += bsum(d); }
    s_cab = c;
    s_sab = sm;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (dstar < 0) {
      // k_selB's range guarantees the answer inside the window
      C.numeric_err = 4;
      J.mode = JM_ALL;
    } else {
      const unsigned kb = lo + ((unsigned)dstar << sh);
      J.cnt_above = s_cab;
      J.sum_above = s_sab;
      if (sh == 0) {                         // single-key buckets: the answer
        if (J.kind == K_L1) {                // entries == kb are inactive
          J.theta = (J.sum_above - J.sigma) / (double)J.cnt_above;
          J.mode = JM_DONE;
        } else {
          J.tau = kb;
          const long long ceq = __ldcg(hc + dstar);
          J.cnt_eq = ceq;
          J.keep_eq = J.k - J.cnt_above;
          J.ties = (J.keep_eq < ceq) ? 1 : 0;
          const double tv = kval(kb);
          J.tau_val2 = tv * tv;
          J.mode = JM_DONE;
        }
      } else {
        const unsigned long long top = (unsigned long long)lo + J.width;
        J.prefix = kb;
        J.width = min(1ull << sh, top - (unsigned long long)kb);
        J.round += 1;
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- k_selB
// w streams through a two-stage shared-memory ring of SB_TILE-chunk tiles
// filled by 1D bulk async copies (cp.async.bulk, mbarrier expect_tx; thread
// 0 issues the next tile before the CTA works on the current one), so the
// loads are decoupled from the per-entry work and from register pressure.
#ifndef SIP_SB_TILE
#define SIP_SB_TILE 2048
#endif
#ifndef SIP_SELB_MINB
#define SIP_SELB_MINB 2
#endif
constexpr int SB_TILE = SIP_SB_TILE;          // chunks (16 B) per stage: 32 KB
__host__ inline size_t selb_smem(int ns = 2) { return (size_t)ns * (SB_TILE + 1) * 16; }

template <class T>
__global__ void __launch_bounds__(BLOCK, SIP_SELB_MINB) k_selB(const __grid_constant__ Prob<T> P) {
  pdl_begin();
  if constexpr (sizeof(T) != 4) return;
  else {
    constexpr int W = VT<T>::W;
    constexpr int PER = SB_TILE / BLOCK;      // chunks per thread per tile
    if (gridDim.x != (unsigned)P.sel_grid) __trap();   // regions are sized for this grid
    Ctrl& C = *P.ctrl;
    if (C.stopped) return;
    extern __shared__ __align__(16) char sb_buf[];
    __shared__ uint64_t bars[SMAX];
    __shared__ SelRange s_rng[MAXJOBS];
    __shared__ unsigned s_cn;
    __shared__ double sh[NWARP + 1];
    __shared__ unsigned f_cnt[FB_N], f_l0[FB_N], f_l1[FB_N];
    const bool check = (C.k % C.opt.check_every) == 0;
    const Geo& g = P.g;
    const int nch = g.N / W;
    const int nj = C.njobs;
    Stage2<1> st;
    const int ns = P.selb_ns;                 // stages: ns - 1 tiles in flight while one is worked on
    st.init(bars, sb_buf, SB_TILE, ns);
    const int lane = threadIdx.x & 31;
    bool any = false;
    for (int jb = 0; jb < nj; ++jb) {
      const Job& J = C.job[jb];
      if (!job_live(J, check)) continue;
      any = true;
      const bool ts = P.sel_tsum && !check && !J.on_s && J.kind == K_L1;   // pass 1's rule
      const SelRange R = range_of_job(J, P.gh_cnt + (size_t)jb * NBUCK, ts ? P.gh_ta + (size_t)jb * NBUCK : nullptr);
      if (threadIdx.x == 0) s_rng[jb] = R;
      __syncthreads();
      double* part = P.partials + ((size_t)blockIdx.x * MAXJOBS + jb) * 3;
      unsigned* cand = P.cand[jb] + (size_t)blockIdx.x * P.cand_per;
      if (R.mode != JM_SEARCH) {
        if (threadIdx.x == 0) { part[0] = 0.0; part[1] = 0.0; part[2] = 0.0; P.ccnt[(size_t)jb * gridDim.x + blockIdx.x] = 0u; }
        continue;
      }
      const SetD<T>& S = P.set[J.set];
      const T* buf = J.on_s ? S.s : S.w;
      const unsigned lo = R.lo, hi = R.hi;
      const int tpb = (nch + SB_TILE - 1) / SB_TILE;              // tiles per operator block
      const int ntile = S.nblk * tpb;
      const int nmine = ntile > (int)blockIdx.x ? (ntile - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
      auto tile_of = [&](int i, int* c0, int* cnt, const T** src) {
        const int t = (int)blockIdx.x + i * (int)gridDim.x;
        const int bl = t / tpb, tt = t - bl * tpb;
        *c0 = tt * SB_TILE;
        *cnt = min(SB_TILE, nch - *c0);
        *src = buf + (int64_t)bl * g.ld + (int64_t)(*c0) * W;
      };
      auto issue = [&](int i) {
        int c0, cnt;
        const T* src;
        tile_of(i, &c0, &cnt, &src);
        const char* sp[1] = {reinterpret_cast<const char*>(src)};
        const unsigned by[1] = {(unsigned)cnt * 16u};
        st.issue(i % ns, 1, sp, by);
      };
      const bool sums = J.kind == K_L1;
      const int fsh = sel_shift((unsigned long long)(hi - lo), FB_BITS);
      if (threadIdx.x == 0) s_cn = 0u;
      for (int d = threadIdx.x; d < FB_N; d += BLOCK) { f_cnt[d] = 0u; f_l0[d] = 0u; f_l1[d] = 0u; }
      __syncthreads();
      unsigned n_ab = 0;                        // per thread: <= the entries it visits
      double s_ab = 0.0;
      const unsigned lo1 = lo > 1u ? lo : 1u;   // zeros are never candidates
      const unsigned wid1 = hi > lo1 ? hi - lo1 : 0u;
      for (int q = 0; q < ns - 1 && q < nmine; ++q) issue(q);
      for (int i = 0; i < nmine; ++i) {
        if (i + ns - 1 < nmine) issue(i + ns - 1);   // the stage worked on at i - 1
        const int sidx = i % ns;
        st.wait(sidx);
        int c0, cnt;
        const T* src;
        tile_of(i, &c0, &cnt, &src);
        const T* tl = reinterpret_cast<const T*>(st.at(sidx, 0));
        unsigned mine = 0;   // candidates of this thread (bit u*W+e)
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int c = u * BLOCK + (int)threadIdx.x;
          T v[W] = {};
          if (c < cnt) VT<T>::ldT_s(tl + c * W, v);     // the tile's tail reads as zeros
#pragma unroll
          for (int e = 0; e < W; ++e) {
            const unsigned k = key32((float)v[e]);
            const bool ab = k >= hi;
            n_ab += ab ? 1u : 0u;
            s_ab += (double)(ab ? __uint_as_float(k) : 0.0f);   // one select + one conversion
            mine |= (unsigned)(k - lo1 < wid1) << (u * W + e);
          }
        }
        // warp-aggregated append to this CTA's region (one shared atomic per warp)
        const int cnt1 = __popc(mine);
        int incl = cnt1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t_ = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t_;
        }
        const int wtot = __shfl_sync(0xffffffffu, incl, 31);
        if (wtot) {
          unsigned base = 0u;
          if (lane == 31) base = atomicAdd(&s_cn, (unsigned)wtot);
          unsigned pos = __shfl_sync(0xffffffffu, base, 31) + (unsigned)(incl - cnt1);
          while (mine) {
            const int bit = __ffs(mine) - 1;
            mine &= mine - 1u;
            const int c = (bit / W) * BLOCK + (int)threadIdx.x;
            const unsigned k = key32((float)tl[c * W + bit % W]);
            cand[pos++] = k;
            const int d = (int)((k - lo) >> fsh);    // the candidates' histogram (counts, limb sums)
            atomicAdd(&f_cnt[d], 1u);
            if (sums) {
              unsigned l[2];
              Limbs<float>::split(k, l);
              atomicAdd(&f_l0[d], l[0]);
              atomicAdd(&f_l1[d], l[1]);
            }
          }
        }
        __syncthreads();   // the stage is refilled by the issue of tile i + ns
      }
      // this CTA's candidate histogram into the job's (non-zero buckets only)
      __syncthreads();
      for (int d = threadIdx.x; d < FB_N; d += BLOCK) {
        if (!f_cnt[d]) continue;
        atomicAdd(P.gf_cnt + (size_t)jb * FB_N + d, f_cnt[d]);
        if (sums) atomicAdd(P.gf_s0 + (size_t)jb * FB_N + d, (unsigned long long)f_l0[d] + ((unsigned long long)f_l1[d] << 16));
      }
      // per-CTA (count, sum above): fixed-order block sums
      const double d_ab = block_sum((double)n_ab, sh);   // exact: counts < 2^53
      const double d_sab = block_sum(s_ab, sh);
      __syncthreads();
      if (threadIdx.x == 0) {
        part[0] = d_ab; part[1] = d_sab; part[2] = 0.0;
        P.ccnt[(size_t)jb * gridDim.x + blockIdx.x] = s_cn;
      }
      __syncthreads();
    }
    if (!any) return;
    if (last_block(P.counter)) {
      for (int jb = 0; jb < nj; ++jb) {
        Job& J = C.job[jb];
        if (!job_live(J, check)) continue;
        const SelRange R = s_rng[jb];
        double tot2[2];
        for (int q = 0; q < 2; ++q) {            // fixed order over the CTAs
          double a = 0.0;
          for (int b = threadIdx.x; b < (int)gridDim.x; b += BLOCK)
            a += __ldcg(P.partials + ((size_t)b * MAXJOBS + jb) * 3 + q);
          tot2[q] = block_sum(a, sh);
        }
        if (threadIdx.x == 0) {
          if (R.mode != JM_SEARCH) {
            J.mode = R.mode;
          } else if (J.kind == K_L1 && C.sums[J.set][J.on_s ? SLOT_FN : SLOT_W2] <= J.sigma) {
            J.mode = JM_INSIDE;                  // ||w||_1 <= sigma (pass 1's sum): w is in the ball (L5)
          } else {
            J.cnt_above = (long long)tot2[0];
            J.sum_above = tot2[1];
            J.prefix = R.lo;                     // the window of the candidates
            J.width = (unsigned long long)(R.hi - R.lo);
            J.round = 1;
          }
        }
        __syncthreads();
        // the candidates' 2^FB_BITS-bucket histogram narrows the window (round 1)
        if (J.mode == JM_SEARCH && J.round == 1)
          resolve_window(C, J, P.gf_cnt + (size_t)jb * FB_N, P.gf_s0 + (size_t)jb * FB_N, FB_BITS);
        for (int d = threadIdx.x; d < NBUCK; d += BLOCK) {   // next round A
          P.gh_cnt[(size_t)jb * NBUCK + d] = 0u;
          P.gh_ta[(size_t)jb * NBUCK + d] = 0ull;
        }
        for (int d = threadIdx.x; d < FB_N; d += BLOCK) {
          P.gf_cnt[(size_t)jb * FB_N + d] = 0u;
          P.gf_s0[(size_t)jb * FB_N + d] = 0ull;
        }
        __syncthreads();
      }
      if (threadIdx.x == 0) *P.counter = 0u;
    }
  }
}

// ---------------------------------------------------------------- k_selC
// One candidate round: this CTA's histogram of the window's keys into the
// job's global histogram; the last CTA resolves the window.  Returns whether
// any job took part (the same answer in every CTA).
template <class T>
__device__ bool selc_round(const Prob<T>& P, Ctrl& C, int round, bool check, unsigned* gen = nullptr) {
  using LB = Limbs<float>;
  __shared__ unsigned h_cnt[NBUCK];
  __shared__ unsigned h_l[LB::N][NBUCK];
  const int nj = C.njobs;
  bool any = false;
  for (int jb = 0; jb < nj; ++jb) {
    const Job& J = C.job[jb];
    if (J.mode != JM_SEARCH || J.round != round || (J.on_s && !check)) continue;
    any = true;
    const bool sums = J.kind == K_L1;
    const unsigned lo = (unsigned)J.prefix;
    const unsigned long long width = J.width;
    const int sh = sel_shift(width, 11);
    for (int d = threadIdx.x; d < NBUCK; d += BLOCK) {
      h_cnt[d] = 0u;
#pragma unroll
      for (int q = 0; q < LB::N; ++q) h_l[q][d] = 0u;
    }
    __syncthreads();
    // this CTA's candidate region (k_selB's CTA of the same index),
    // coalesced, eight loads in flight per thread; only the window's keys
    // (a small part after k_selB's round) reach the shared histogram
    const unsigned* cand = P.cand[jb] + (size_t)blockIdx.x * P.cand_per;
    const int n = (int)__ldcg(P.ccnt + (size_t)jb * gridDim.x + blockIdx.x);
    for (int qb = 0; qb < n; qb += BLOCK * 8) {
      unsigned kk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int q = qb + u * BLOCK + (int)threadIdx.x;
        kk[u] = q < n ? __ldcg(cand + q) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned k = kk[u];
        if (qb + u * BLOCK + (int)threadIdx.x >= n || k < lo || (unsigned long long)(k - lo) >= width) continue;
        const int d = (int)((k - lo) >> sh);
        atomicAdd(&h_cnt[d], 1u);
        if (sums) {
          unsigned l[LB::N];
          LB::split(k, l);
#pragma unroll
          for (int t = 0; t < LB::N; ++t) atomicAdd(&h_l[t][d], l[t]);
        }
      }
    }
    __syncthreads();
    unsigned* gc = P.gh_cnt + (size_t)jb * NBUCK;
    unsigned long long* g0 = P.gh_s0 + (size_t)jb * NBUCK;
    for (int d = threadIdx.x; d < NBUCK; d += BLOCK) {
      if (!h_cnt[d]) continue;
      atomicAdd(gc + d, h_cnt[d]);
      if (sums) atomicAdd(g0 + d, (unsigned long long)h_l[0][d] + ((unsigned long long)h_l[1][d] << 16));
    }
    __syncthreads();
  }
  if (!any) return false;
  if (last_block(P.counter)) {
    for (int jb = 0; jb < nj; ++jb) {
      Job& J = C.job[jb];
      if (J.mode != JM_SEARCH || J.round != round || (J.on_s && !check)) continue;
      resolve_window(C, J, P.gh_cnt + (size_t)jb * NBUCK, P.gh_s0 + (size_t)jb * NBUCK, 11);
      for (int d = threadIdx.x; d < NBUCK; d += BLOCK) {
        P.gh_cnt[(size_t)jb * NBUCK + d] = 0u;
        P.gh_s0[(size_t)jb * NBUCK + d] = 0ull;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      if (gen) { __threadfence(); atomicAdd(gen, 1u); }   // release the round (k_selCF)
    }
  }
  return true;
}

template <class T>
__global__ void __launch_bounds__(BLOCK) k_selC(const __grid_constant__ Prob<T> P, int round) {
  pdl_begin();
  if constexpr (sizeof(T) != 4) return;
  else {
    if (gridDim.x != (unsigned)P.sel_grid) __trap();   // one CTA per k_selB region
    Ctrl& C = *P.ctrl;
    if (C.stopped) return;
    selc_round(P, C, round, (C.k % C.opt.check_every) == 0);
  }
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// The candidate rounds 2..4 in one launch: between rounds every CTA waits
// for the last CTA's window (a release counter that only ever grows, read by
// each CTA before its first arrival, so no reset races).  The grid is one
// resident wave (k_selB's), and the next kernel launches only after all of
// this grid's CTAs run (PDL), so the spin cannot starve a CTA of a slot.
template <class T>
__global__ void __launch_bounds__(BLOCK) k_selCF(const __grid_constant__ Prob<T> P) {
  pdl_begin();
  if constexpr (sizeof(T) != 4) return;
  else {
    if (gridDim.x != (unsigned)P.sel_grid) __trap();
    Ctrl& C = *P.ctrl;
    if (C.stopped) return;
    __shared__ unsigned s_base;
    if (threadIdx.x == 0) s_base = ld_acquire(P.sel_gen);
    __syncthreads();
    const unsigned base = s_base;
    const bool check = (C.k % C.opt.check_every) == 0;
    unsigned nb = 0;
    for (int round = 2; round <= 4; ++round) {
      if (!selc_round(P, C, round, check, P.sel_gen)) break;   // no job left (every CTA agrees)
      ++nb;
      // the last CTA bumps sel_gen once its window is written; wait for it
      if (threadIdx.x == 0) {
        while ((int)(ld_acquire(P.sel_gen) - base) < (int)nb) __nanosleep(32);
        __threadfence();
      }
      __syncthreads();
    }
  }
}

// SIP_SEL_DEBUG=1: the jobs after the threshold search (diagnostics)
template <class T>
__global__ void k_seldbg(const __grid_constant__ Prob<T> P) {
  const Ctrl& C = *P.ctrl;
  if (threadIdx.x || blockIdx.x || C.stopped) return;
  for (int jb = 0; jb < C.njobs; ++jb) {
    const Job& J = C.job[jb];
    unsigned long long ncand = 0;   // k_selB's candidates (select v2 only)
    if (P.selv2)
      for (int b = 0; b < P.sel_grid; ++b) ncand += P.ccnt[(size_t)jb * P.sel_grid + b];
    printf("k=%d job=%d on_s=%d kind=%d mode=%d round=%d theta=%.17g tau=%llu cnt_above=%lld sum_above=%.17g prefix=%llu width=%llu keep_eq=%lld ties=%d ncand=%llu\n",
           C.k, jb, J.on_s, J.kind, J.mode, J.round, J.theta, J.tau, J.cnt_above, J.sum_above, J.prefix, J.width,
           J.keep_eq, J.ties, ncand);
  }
}

}  // namespace sip
