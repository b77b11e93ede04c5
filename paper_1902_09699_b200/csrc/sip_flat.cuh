// sip_flat.cuh -- flattened, vectorised set passes (sm_100a).
//
// The per-set work of Algorithm 1 is independent per set and per
// entry, so instead of looping over the sets inside a thread, the iteration
// space is flattened into segments: segment 0 = the per-point x work (x
// history, Alg. 2 snapshot of x, Eq. 27 norms), then one segment per
// (set, operator block).  A warp takes 32 consecutive W-point chunks of one
// segment, so every branch is warp-uniform, registers stay low (high
// occupancy) and each lane issues all its 16-byte loads before computing.
// k_pass2f uses CTA-wide tiles of BLOCK chunks (the cardinality tie rank is
// a block scan); k_tiecountf uses the same tiles.
#pragma once
#include "sip_vec.cuh"

namespace sip {

// A_prim x on a chunk (Eq. 8), with the x row loaded by the caller
template <class T>
__device__ __forceinline__ void prim_chunk(const Geo& g, int prim, const T* x, int pt0, int lane,
                                           const Loc& L, const double* xc, double* s) {
  constexpr int W = VT<T>::W;
  if (prim == PRIM_I) {
#pragma unroll
    for (int e = 0; e < W; ++e) s[e] = xc[e];
  } else if (prim == PRIM_X) {
    double xr = __shfl_down_sync(0xffffffffu, xc[0], 1);
    if (lane == 31) xr = (double)x[pt0 + W];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const double nx_ = e < W - 1 ? xc[e + 1] : xr;
      s[e] = (L.ix + e < g.nx - 1) ? (nx_ - xc[e]) * g.ihx : 0.0;
    }
  } else {
    const bool z = prim == PRIM_Z;
    double t[W];
    VT<T>::ld(x + pt0 + (z ? g.plane : g.nx), t);
    const bool hi = z ? (L.gz < g.nz_g - 1) : (L.iy < g.ny - 1);
    const double ih = z ? g.ihz : g.ihy;
#pragma unroll
    for (int e = 0; e < W; ++e) s[e] = hi ? (t[e] - xc[e]) * ih : 0.0;
  }
}

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

template <class T>
__global__ void __launch_bounds__(BLOCK, 2) k_pass1f(const __grid_constant__ Prob<T> P) {
  constexpr int W = VT<T>::W;
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
  const int nch = g.N / W;
  const int gps = (nch + 31) >> 5;                       // warp groups per segment
  const int lane = threadIdx.x & 31;
  const int total = P.nseg1 * gps;
  for (int grp = blockIdx.x * NWARP + (threadIdx.x >> 5); grp < total; grp += gridDim.x * NWARP) {
    const int seg = grp / gps;
    const int c = (grp - seg * gps) * 32 + lane;
    const bool valid = c < nch;
    const int pt0 = (valid ? c : nch - 1) * W;
    const Loc L = locate(g, pt0);
    double xc[W];
    VT<T>::ld(P.x + pt0, xc);
    if (seg == 0) {
      // x history (Eq. 27) and Alg. 2's x snapshot
      if (check) {
        T h[HIST_S][W];
#pragma unroll
        for (int js = 0; js < HIST_S; ++js)      // physical slots; valid ones are the
          if ((hhead - js + HIST_S) % HIST_S < hcount)   // hcount newest
            VT<T>::ldT(P.hist[js] + pt0, h[js]);
        double x2 = 0.0;
#pragma unroll
        for (int e = 0; e < W; ++e) x2 += valid ? xc[e] * xc[e] : 0.0;
        warp_acc(acc, nv, P.P * NSLOT, x2);
#pragma unroll
        for (int js = 0; js < HIST_S; ++js) {
          if ((hhead - js + HIST_S) % HIST_S >= hcount) continue;
          double d2 = 0.0;
#pragma unroll
          for (int e = 0; e < W; ++e) {
            const double d = xc[e] - (double)h[js][e];
            d2 += valid ? d * d : 0.0;
          }
          warp_acc(acc, nv, P.P * NSLOT + 1 + js, d2);
        }
      }
      if (valid) {
        VT<T>::st(P.hist[hslot] + pt0, xc);
        if (adapt) VT<T>::st(xs_wr + pt0, xc);
      }
      continue;
    }
    const int i = P.seg_set[seg], bl = P.seg_blk[seg];
    const SetD<T>& S = P.set[i];
    const int prim = S.prim[bl];
    const int64_t off = (int64_t)bl * g.ld + pt0;
    const bool pointwise = (S.kind == K_BOUNDS || S.kind == K_DIST);
    // issue every load of the chunk first
    T yo[W], vo[W], lo[W], hi[W], mm[W], y0[W], v0[W], vh0[W];
    VT<T>::ldT(S.y[par] + off, yo);
    VT<T>::ldT(S.v[par] + off, vo);
    if (S.lo_vec) VT<T>::ldT(S.lo_vec + off, lo);
    if (S.hi_vec) VT<T>::ldT(S.hi_vec + off, hi);
    if (S.kind == K_DIST) VT<T>::ldT(P.m + pt0, mm);
    if (dots) {
      VT<T>::ldT(S.vh0 + off, vh0);
      if (pointwise) {
        VT<T>::ldT(S.y[par ^ 1] + off, y0);
        VT<T>::ldT(S.v[par ^ 1] + off, v0);
      }
    }
    double s[W], s0[W];
    prim_chunk<T>(g, prim, P.x, pt0, lane, L, xc, s);
    if (dots) {
      double xo[W];
      VT<T>::ld(xs_rd + pt0, xo);
      prim_chunk<T>(g, prim, xs_rd, pt0, lane, L, xo, s0);
    }
    // per-point arithmetic in the storage precision T (reading L20); the
    // reductions are summed per chunk in T and accumulated in fp64
    const T rho = (T)C.rho[i], gam = (T)C.gamma[i], one = (T)1;
    const T irho = (T)(1.0 / C.rho[i]), i1rho = (T)(1.0 / (1.0 + C.rho[i]));
    const T tlo = (T)S.lo, thi = (T)S.hi;
    T a_w2 = 0, a_hv = 0, a_hh = 0, a_vh = 0, a_gv = 0, a_gg = 0, a_vv = 0, a_fn = 0, a_s2 = 0;
    T yn[W], vn[W], wv[W], vh[W], st_s[W];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const bool pad = !valid || pad_vec(g, prim, L, e);
      const T sv = pad ? (T)0 : (T)s[e];
      st_s[e] = sv;
      const T xbar = gam * sv + (one - gam) * yo[e];                // relaxation
      // fp64 keeps the exact divisions of the oracle; fp32 uses reciprocals
      const T w = xbar - (sizeof(T) == 8 ? vo[e] / rho : vo[e] * irho);
      wv[e] = pad ? (T)0 : w;
      if (pointwise) {
        T y;
        if (S.kind == K_DIST) {
          y = sizeof(T) == 8 ? (mm[e] + rho * w) / (one + rho) : (mm[e] + rho * w) * i1rho;   // Eq. 22
        } else {
          const T l = S.lo_vec ? lo[e] : tlo;
          const T h = S.hi_vec ? hi[e] : thi;
          y = w < l ? l : (w > h ? h : w);                          // box clamp
          if (check && !pad) {
            const T cl = sv < l ? l : (sv > h ? h : sv);
            a_fn += (sv - cl) * (sv - cl);
          }
        }
        const T vt = rho * (y - w);                                 // Eq. 21 as rho (y - w), L26
        yn[e] = pad ? (T)0 : y;
        vn[e] = pad ? (T)0 : vt;
        if (dots && !pad) {
          const T dg = y0[e] - y;
          const T dv = vt - v0[e];
          a_gv += dg * dv; a_gg += dg * dg; a_vv += dv * dv;
        }
      } else if (!pad) {
        a_w2 += w * w;
      }
      if (adapt) {                                                  // Alg. 2 line 1
        const T vht = vo[e] + rho * (yo[e] - sv);
        vh[e] = pad ? (T)0 : vht;
        if (dots && !pad) {
          const T dvh = vht - vh0[e];
          const T dh = sv - (T)s0[e];
          a_hv += dh * dvh; a_hh += dh * dh; a_vh += dvh * dvh;
        }
      }
      if (check && !pad) a_s2 += sv * sv;
    }
    if (valid) {
      if (pointwise) {
        VT<T>::stT(S.y[par ^ 1] + off, yn);
        VT<T>::stT(S.v[par ^ 1] + off, vn);
      } else {
        VT<T>::stT(S.w + off, wv);
        if (check && S.s) VT<T>::stT(S.s + off, st_s);
      }
      if (adapt) VT<T>::stT(S.vh0 + off, vh);
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
  double* stage = P.partials + (size_t)gridDim.x * nv;
  if (finish_reduction(acc, nv, P.partials, P.counter, stage, sh)) {
    for (int v = threadIdx.x; v < nv; v += BLOCK) {
      const double val = __ldcg(stage + v);
      if (v < P.P * NSLOT) C.sums[v / NSLOT][v % NSLOT] = val;
      else C.evol[v - P.P * NSLOT] = val;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < P.P; ++i) {   // l2 / annulus radial factors (Table 1, L7)
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

template <class T>
__global__ void __launch_bounds__(BLOCK) k_pass2f(const __grid_constant__ Prob<T> P) {
  using K = KeyT<T>;
  using U = typename K::U;
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  extern __shared__ double acc[];
  __shared__ double sh[NWARP + 1];
  __shared__ int s_w[NWARP];
  const Geo& g = P.g;
  const int nv = P.P * 4;
  const int k = C.k, par = k & 1;
  const bool adapt = is_adapt_it(k, C.opt.adapt_every);
  const bool dots = adapt && C.first_adapt_done;
  const bool check = (k % C.opt.check_every) == 0;
  for (int v = threadIdx.x; v < NWARP * nv; v += BLOCK) acc[v] = 0.0;
  __syncthreads();
  const int nch = g.N / W;
  const int tpb = (nch + BLOCK - 1) / BLOCK;
  const int total = P.nseg2 * tpb;
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int sg = t / tpb, lt = t - sg * tpb;
    const int i = P.seg2_set[sg], bl = P.seg2_blk[sg];
    const SetD<T>& S = P.set[i];
    const int prim = S.prim[bl];
    const int c = lt * BLOCK + threadIdx.x;
    const bool valid = c < nch;
    const int pt0 = (valid ? c : nch - 1) * W;
    const Loc L = locate(g, pt0);
    const int64_t off = (int64_t)bl * g.ld + pt0;
    T wv[W], y0[W], v0[W];
    VT<T>::ldT(S.w + off, wv);
    if (dots) {
      VT<T>::ldT(S.y[par ^ 1] + off, y0);
      VT<T>::ldT(S.v[par ^ 1] + off, v0);
    }
    const double rho = C.rho[i];
    bool pad[W];
#pragma unroll
    for (int e = 0; e < W; ++e) pad[e] = !valid || pad_vec(g, prim, L, e);
    double y[W];
    if (S.kind == K_L1) {
      const Job& J = C.job[S.job];
#pragma unroll
      for (int e = 0; e < W; ++e) {
        const double w = (double)wv[e];
        if (J.mode == JM_DONE) {
          const double a = fabs(w) - J.theta;
          y[e] = a > 0.0 ? (w > 0.0 ? a : -a) : 0.0;   // soft threshold
        } else {
          y[e] = (J.mode == JM_INSIDE || J.mode == JM_ALL) ? w : 0.0;
        }
      }
    } else if (S.kind == K_CARD) {
      const Job& J = C.job[S.job];
      bool keep[W];
      int cnt = 0;
#pragma unroll
      for (int e = 0; e < W; ++e) {
        const U key = K::key(wv[e]);
        keep[e] = (J.mode == JM_ALL) || (J.mode == JM_DONE && key > (U)J.tau);
        cnt += (J.mode == JM_DONE && !pad[e] && key == (U)J.tau) ? 1 : 0;
      }
      if (J.mode == JM_DONE) {
        if (J.ties) {   // the first keep_eq entries == tau in index order (L6)
          const int* toff = P.tiecnt + (size_t)S.job * P.ntiles_max;
          long long r = (long long)toff[bl * tpb + lt] + block_excl_count(cnt, s_w);
#pragma unroll
          for (int e = 0; e < W; ++e)
            if (!pad[e] && K::key(wv[e]) == (U)J.tau) { if (r < J.keep_eq) keep[e] = true; ++r; }
        } else {
#pragma unroll
          for (int e = 0; e < W; ++e) if (K::key(wv[e]) == (U)J.tau) keep[e] = true;
        }
      }
#pragma unroll
      for (int e = 0; e < W; ++e) y[e] = keep[e] ? (double)wv[e] : 0.0;
    } else {   // l2 ball / annulus radial scaling (L7 at 0)
      const double sc = C.ann_scale[i];
      const int az = C.ann_zero[i];
#pragma unroll
      for (int e = 0; e < W; ++e)
        y[e] = az ? ((bl == 0 && pt0 + e == S.first_real) ? C.sig_lo[i] : 0.0) : (double)wv[e] * sc;
    }
    T yn[W], vn[W];
    double a_gv = 0, a_gg = 0, a_vv = 0;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const double yt = pad[e] ? 0.0 : (double)(T)y[e];
      const double vt = pad[e] ? 0.0 : (double)(T)(rho * (yt - (double)wv[e]));
      yn[e] = (T)yt;
      vn[e] = (T)vt;
      if (dots && !pad[e]) {
        const double dg = -(yt - (double)y0[e]);
        const double dv = vt - (double)v0[e];
        a_gv += dg * dv; a_gg += dg * dg; a_vv += dv * dv;
      }
    }
    if (valid) {
      VT<T>::stT(S.y[par ^ 1] + off, yn);
      VT<T>::stT(S.v[par ^ 1] + off, vn);
    }
    if (dots) {
      warp_acc(acc, nv, i * 4 + 0, a_gv);
      warp_acc(acc, nv, i * 4 + 1, a_gg);
      warp_acc(acc, nv, i * 4 + 2, a_vv);
    }
  }
  // Eq. 26 numerators of l1 / cardinality sets from s (check iterations)
  if (check) {
    for (int i = 0; i < P.P; ++i) {
      const SetD<T>& S = P.set[i];
      if (!S.global || S.sjob < 0) continue;
      const Job& Js = C.job[S.sjob];
      double fn = 0.0;
      if (Js.mode == JM_DONE) {
        const int tot = S.nblk * nch;
        for (int q = blockIdx.x * BLOCK + threadIdx.x; q < tot; q += gridDim.x * BLOCK) {
          const int bl = (q >= nch) + (q >= 2 * nch), c = q - bl * nch;   // nblk <= 3
          T sv[W];
          VT<T>::ldT(S.s + (int64_t)bl * g.ld + (int64_t)c * W, sv);
#pragma unroll
          for (int e = 0; e < W; ++e) {
            const double v = (double)sv[e];
            if (S.kind == K_L1) {
              const double a = fabs(v) < Js.theta ? fabs(v) : Js.theta;
              fn += a * a;
            } else if (K::key(sv[e]) < (U)Js.tau) {
              fn += v * v;
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

}  // namespace sip
