// sip_flat.cuh -- the exact radix threshold search over the flattened
// (set, block) segments of the global sets (sm_100a): k_selectf (the l1-ball
// threshold and the cardinality k-th key, readings L5/L6) and
// k_tiecountf (index-order tie offsets of the top-k, L6).  A CTA tile is
// BLOCK consecutive W-point chunks of one segment, so every branch is
// warp-uniform; the tie rank is a block scan (block_excl_count).
#pragma once
#include "sip_vec.cuh"

namespace sip {

// exclusive rank of this thread's flags within the CTA tile (fixed order:
// warps in order, lanes in order, elements in order)
__device__ __forceinline__ int block_excl_count(int cnt, int* s_w) {
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  int inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_w[wp] = inc;
  __syncthreads();
  int before = 0;
  for (int q = 0; q < wp; ++q) before += s_w[q];
  __syncthreads();
  return before + inc - cnt;
}

// ------------------------------------------------------------ select (vectorised)
// Histograms use native 32-bit shared atomics only (64-bit shared atomic add
// compiles to a CAS spin loop): the significand is split into 16-bit limbs
// whose per-CTA sums are flushed to 64-bit global atomics every SEL_FLUSH
// elements (so no 32-bit limb sum can overflow).  Counts and sums stay exact
// integers, so the result is independent of the accumulation order.
constexpr int SEL_U = 4;                           // chunks in flight per thread
constexpr int SEL_FLUSH_IT = 65536 / (BLOCK * 4 * SEL_U);   // iterations between flushes

template <class T> struct Limbs;
template <> struct Limbs<float> {
  static constexpr int N = 2;                      // 24-bit significand: 16 + 8 bits
  __device__ static void split(uint32_t key, unsigned* l) {
    const uint32_t e = key >> 23, m = key & 0x7fffffu;
    const uint32_t sig = (e ? (1u << 23) : 0u) | m;
    l[0] = sig & 0xffffu; l[1] = sig >> 16;
  }
};
template <> struct Limbs<double> {
  static constexpr int N = 4;                      // 53-bit significand: 4 x 16 bits
  __device__ static void split(unsigned long long key, unsigned* l) {
    const unsigned long long e = key >> 52, m = key & 0xfffffffffffffull;
    const unsigned long long sig = (e ? (1ull << 52) : 0ull) | m;
    l[0] = (unsigned)(sig & 0xffffu); l[1] = (unsigned)((sig >> 16) & 0xffffu);
    l[2] = (unsigned)((sig >> 32) & 0xffffu); l[3] = (unsigned)(sig >> 48);
  }
};

// multi-rank: a job's histogram in the gather slot, HJOB doubles per job:
// sums s0, s1 (u64 x NBUCK each), then the counts (u32 x NBUCK)
constexpr int HJOB = NBUCK * 2 + NBUCK / 2;
template <class T>
__device__ inline void publish_hist(const Prob<T>& P, int jb, const unsigned* gc, const unsigned long long* g0,
                                    const unsigned long long* g1) {
  double* base = P.xg + (size_t)P.rank * P.xslot + (size_t)jb * HJOB;
  unsigned long long* s0 = reinterpret_cast<unsigned long long*>(base);
  unsigned long long* s1 = s0 + NBUCK;
  unsigned* cn = reinterpret_cast<unsigned*>(s1 + NBUCK);
  for (int d = threadIdx.x; d < NBUCK; d += blockDim.x) {
    s0[d] = __ldcg(g0 + d); s1[d] = __ldcg(g1 + d); cn[d] = __ldcg(gc + d);
  }
}

template <class T>
__global__ void __launch_bounds__(BLOCK) k_selectf(const __grid_constant__ Prob<T> P, int round) {
  pdl_begin();
  using K = KeyT<T>;
  using U = typename K::U;
  using LB = Limbs<T>;
  constexpr int W = VT<T>::W;
  // the per-CTA candidate regions (cand_per) and the ccnt stride are sized
  // for this grid: any other launch geometry would overrun them
  if (gridDim.x != (unsigned)P.sel_grid) __trap();
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  __shared__ unsigned h_cnt[NBUCK];
  __shared__ unsigned h_l[LB::N][NBUCK];
  __shared__ unsigned s_cn;   // candidates appended by this CTA (round 2)
  const Geo& g = P.g;
  const bool check = (C.k % C.opt.check_every) == 0;
  int lo, nb, plo = 0, pnb = 0;
  digit_bits(K::BITS, round, &lo, &nb);
  if (round > 1) digit_bits(K::BITS, round - 1, &plo, &pnb);
  const U dmask = (U)((1u << nb) - 1u);
  const int nbk = 1 << nb;
  const int nch = g.N / W;
  bool any = false;
  for (int jb = 0; jb < C.njobs; ++jb) {
    const Job& J = C.job[jb];
    if (J.mode != JM_SEARCH || J.round != round - 1 || (J.on_s && !check)) continue;
    any = true;
    unsigned* gc = P.gh_cnt + (size_t)jb * NBUCK;
    unsigned long long* g0 = P.gh_s0 + (size_t)jb * NBUCK;
    unsigned long long* g1 = P.gh_s1 + (size_t)jb * NBUCK;
    const SetD<T>& S = P.set[J.set];
    const T* buf = J.on_s ? S.s : S.w;
    const U prefix = (U)J.prefix;
    const bool sums = (J.kind == K_L1);
    const int tot = S.nblk * nch;
    auto clear = [&]() {
      for (int d = threadIdx.x; d < nbk; d += BLOCK) {
        h_cnt[d] = 0u;
#pragma unroll
        for (int q = 0; q < LB::N; ++q) h_l[q][d] = 0u;
      }
    };
    auto flush = [&]() {
      __syncthreads();
      for (int d = threadIdx.x; d < nbk; d += BLOCK) {
        if (h_cnt[d] == 0u) continue;
        atomicAdd(gc + d, h_cnt[d]);
        if (sums) {
          unsigned long long s0 = (unsigned long long)h_l[0][d] + ((unsigned long long)h_l[1][d] << 16);
          atomicAdd(g0 + d, s0);
          if (LB::N > 2) {
            unsigned long long s1 = (unsigned long long)h_l[LB::N > 2 ? 2 : 0][d] +
                                    ((unsigned long long)h_l[LB::N > 3 ? 3 : 0][d] << 16);
            if (s1) atomicAdd(g1 + d, s1);
          }
        }
      }
      __syncthreads();
      clear();
      __syncthreads();
    };
    clear();
    if (threadIdx.x == 0) s_cn = 0u;
    __syncthreads();
    const int stride = gridDim.x * BLOCK * SEL_U;
    int it = 0;
    // fp32 candidate compaction: round 2 appends the keys of the round-1
    // bucket (its survivors), rounds >= 3 read only those
    // each CTA appends to its own region (a shared counter, no global
    // contention) and round >= 3 reads back its own region: rounds 2 and 3
    // run on the same grid
    unsigned* cand = (sizeof(T) == 4) ? P.cand[jb] + (size_t)blockIdx.x * P.cand_per : nullptr;
    const bool make_cand = cand && round == 2;
    const bool use_cand = cand && round >= 3;
    unsigned* ccnt = P.ccnt + (size_t)jb * gridDim.x + blockIdx.x;
    const int ntot = use_cand ? (int)__ldcg(ccnt) : tot;
    auto hkey = [&](U key) {   // one shared reduction per entry and counter (measured faster than run merging)
      const int d = (int)((key >> lo) & dmask);
      atomicAdd(&h_cnt[d], 1u);
      if (sums) {
        unsigned l[LB::N];
        LB::split(key, l);
#pragma unroll
        for (int q = 0; q < LB::N; ++q) atomicAdd(&h_l[q][d], l[q]);
      }
    };
    // block-uniform trip count (the periodic flush synchronises the CTA)
    const int b_first = use_cand ? 0 : blockIdx.x * BLOCK * SEL_U;
    const int b_step = use_cand ? BLOCK * SEL_U : stride;
    for (int b0 = b_first; b0 < ntot; b0 += b_step) {
      const int q0 = b0 + threadIdx.x;
      if (use_cand) {
        U kk[SEL_U];
        bool ok[SEL_U];
#pragma unroll
        for (int u = 0; u < SEL_U; ++u) {
          const int q = q0 + u * BLOCK;
          ok[u] = q < ntot;
          kk[u] = ok[u] ? (U)__ldcg(cand + q) : (U)0;
        }
#pragma unroll
        for (int u = 0; u < SEL_U; ++u)
          if (ok[u] && (U)(kk[u] >> plo) == prefix) hkey(kk[u]);
      } else {
        T v[SEL_U][W];
        bool ok[SEL_U];
#pragma unroll
        for (int u = 0; u < SEL_U; ++u) {   // all loads of the iteration first
          const int q = q0 + u * BLOCK;
          ok[u] = q < tot;
          const int qq = ok[u] ? q : tot - 1;
          const int bl = (qq >= nch) + (qq >= 2 * nch);   // nblk <= 3: no integer division
          VT<T>::ldT(buf + (int64_t)bl * g.ld + (int64_t)(qq - bl * nch) * W, v[u]);
        }
        unsigned mine = 0;   // survivors of this thread (bit u*W+e)
#pragma unroll
        for (int u = 0; u < SEL_U; ++u) {
#pragma unroll
          for (int e = 0; e < W; ++e) {
            const U key = K::key(v[u][e]);
            const bool in = ok[u] && (round == 1 || (U)(key >> plo) == prefix);
            if (in) { hkey(key); mine |= 1u << (u * W + e); }
          }
        }
        if (make_cand) {   // warp-aggregated append: one global atomic per warp, no block barrier
          const int lane = threadIdx.x & 31;
          const int cnt = __popc(mine);
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t_ = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t_;
          }
          const int tot_ = __shfl_sync(0xffffffffu, incl, 31);
          unsigned base_ = 0u;
          if (lane == 31 && tot_ > 0) base_ = atomicAdd(&s_cn, (unsigned)tot_);
          unsigned pos = __shfl_sync(0xffffffffu, base_, 31) + (unsigned)(incl - cnt);
#pragma unroll
          for (int u = 0; u < SEL_U; ++u)
#pragma unroll
            for (int e = 0; e < W; ++e)
              if (mine & (1u << (u * W + e))) cand[pos++] = (unsigned)K::key(v[u][e]);
        }
      }
      if (++it == SEL_FLUSH_IT) { it = 0; flush(); }
    }
    flush();
    if (make_cand && threadIdx.x == 0) *ccnt = s_cn;
  }
  if (!any) return;
  if (last_block(P.counter)) {
    for (int jb = 0; jb < C.njobs; ++jb) {
      Job& J = C.job[jb];
      if (J.mode != JM_SEARCH || J.round != round - 1 || (J.on_s && !check)) continue;
      unsigned* gc = P.gh_cnt + (size_t)jb * NBUCK;
      unsigned long long* g0 = P.gh_s0 + (size_t)jb * NBUCK;
      unsigned long long* g1 = P.gh_s1 + (size_t)jb * NBUCK;
      if (P.nranks > 1) publish_hist(P, jb, gc, g0, g1);
      else resolve_round<T>(P, J, round, gc, g0, g1);
      __syncthreads();
      for (int d = threadIdx.x; d < NBUCK; d += BLOCK) { gc[d] = 0u; g0[d] = 0ull; g1[d] = 0ull; }
      __syncthreads();
    }
    if (threadIdx.x == 0) *P.counter = 0u;
  }
}

// ------------------------------------------------------------ ties / pass2 (CTA tiles)
template <class T>
__global__ void __launch_bounds__(BLOCK) k_tiecountf(const __grid_constant__ Prob<T> P) {
  pdl_begin();
  using K = KeyT<T>;
  using U = typename K::U;
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  __shared__ int s_w[NWARP];
  __shared__ long long s_c[BLOCK];
  __shared__ double s_sh[NWARP + 1];
  const Geo& g = P.g;
  const int nch = g.N / W;
  const int tpb = (nch + BLOCK - 1) / BLOCK;
  bool any = false;
  for (int i = 0; i < P.P; ++i) {
    const SetD<T>& S = P.set[i];
    if (S.kind != K_CARD || S.job < 0) continue;
    const Job& J = C.job[S.job];
    if (J.mode != JM_DONE || !J.ties) continue;
    any = true;
    int* tc = P.tiecnt + (size_t)S.job * P.ntiles_max;
    const int nt = S.nblk * tpb;
    for (int t = blockIdx.x; t < nt; t += gridDim.x) {
      const int bl = t / tpb, c = (t - bl * tpb) * BLOCK + threadIdx.x;
      int cnt = 0;
      if (c < nch) {
        T v[W];
        VT<T>::ldT(S.w + (int64_t)bl * g.ld + (int64_t)c * W, v);
#pragma unroll
        for (int e = 0; e < W; ++e) cnt += (K::key(v[e]) == (U)J.tau) ? 1 : 0;
      }
      const int before = block_excl_count(cnt, s_w);
      if (threadIdx.x == BLOCK - 1) tc[t] = before + cnt;
    }
  }
  if (!any) return;
  if (last_block(P.counter)) {
    for (int i = 0; i < P.P; ++i) {
      const SetD<T>& S = P.set[i];
      if (S.kind != K_CARD || S.job < 0) continue;
      const Job& J = C.job[S.job];
      if (J.mode != JM_DONE || !J.ties) continue;
      int* tc = P.tiecnt + (size_t)S.job * P.ntiles_max;
      const int nt = S.nblk * tpb;
      if (P.nranks > 1)   // this rank's ties per block, for the cross-rank offsets (k_fin)
        for (int bl = 0; bl < S.nblk; ++bl) {
          double c = 0.0;
          for (int t = bl * tpb + threadIdx.x; t < (bl + 1) * tpb; t += BLOCK) c += (double)__ldcg(tc + t);
          c = block_sum(c, s_sh);
          if (threadIdx.x == 0) P.xg[(size_t)P.rank * P.xslot + i * 3 + bl] = c;
        }
      const int per = (nt + BLOCK - 1) / BLOCK;
      const int t0 = threadIdx.x * per;
      long long loc = 0;
      for (int t = t0; t < t0 + per && t < nt; ++t) loc += __ldcg(tc + t);
      s_c[threadIdx.x] = loc;
      __syncthreads();
      if (threadIdx.x == 0) {
        long long run = 0;
        for (int t = 0; t < BLOCK; ++t) { long long cc = s_c[t]; s_c[t] = run; run += cc; }
      }
      __syncthreads();
      long long run = s_c[threadIdx.x];
      for (int t = t0; t < t0 + per && t < nt; ++t) {
        const int cc = __ldcg(tc + t);
        tc[t] = (int)run;
        run += cc;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) *P.counter = 0u;
  }
}

}  // namespace sip
