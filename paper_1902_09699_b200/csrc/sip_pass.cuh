// sip_pass.cuh -- specialised set passes of Algorithm 1 (sm_100a).
//
// k_pass1t / k_pass2t are k_pass1f / k_pass2f with the iteration type fixed
// at graph-capture time: the pattern of adapt iterations (mod(k, 2) = 1,
// P:291) and stop checks (every 5th) repeats every 10 iterations, so
// a captured graph of 10 iterations knows, for each launch, whether Alg. 2's
// inner products and the Eq. 26/27 statistics are needed (template values
// AD, CK in {0, 1}; 2 = decide at run time from the control block).  Inside,
// each (set, block) segment dispatches on the set kind to a body compiled
// for that kind only, so no thread executes predicated code of other kinds.
// Per-point arithmetic is in the storage type T; every reduction is
// accumulated in fp64 (reading L20).
#pragma once
#include "sip_flat.cuh"

namespace sip {

struct IterFlags { bool adapt, dots, check; };

template <int AD, int CK>
__device__ __forceinline__ IterFlags iter_flags(Ctrl& C) {
  const int k = C.k;
  const bool ad = is_adapt_it(k, C.opt.adapt_every);
  const bool ck = (k % C.opt.check_every) == 0;
  if (AD != 2 || CK != 2) {   // the captured variant must match the device iteration
    if (threadIdx.x == 0 && blockIdx.x == 0 &&
        ((AD != 2 && ad != (AD == 1)) || (CK != 2 && ck != (CK == 1))))
      C.numeric_err = 3;
  }
  IterFlags f;
  f.adapt = AD == 2 ? ad : (AD == 1);
  f.check = CK == 2 ? ck : (CK == 1);
  f.dots = f.adapt && C.first_adapt_done;
  return f;
}

// A_prim x on a chunk in the storage precision (Eq. 8; pads -> 0)
template <class T>
__device__ __forceinline__ void prim_chunkT(const Geo& g, int prim, const T* x, int pt0, int lane,
                                            const Loc& L, const T* xc, T* s) {
  constexpr int W = VT<T>::W;
  if (prim == PRIM_I) {
#pragma unroll
    for (int e = 0; e < W; ++e) s[e] = xc[e];
  } else if (prim == PRIM_X) {
    T xr = __shfl_down_sync(0xffffffffu, xc[0], 1);
    if (lane == 31) xr = x[pt0 + W];
    const T ih = (T)g.ihx;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const T nx_ = e < W - 1 ? xc[e + 1] : xr;
      s[e] = (L.ix + e < g.nx - 1) ? (nx_ - xc[e]) * ih : (T)0;
    }
  } else {
    const bool z = prim == PRIM_Z;
    T t[W];
    VT<T>::ldT(x + pt0 + (z ? g.plane : g.nx), t);
    const bool hi = z ? (L.gz < g.nz_g - 1) : (L.iy < g.ny - 1);
    const T ih = (T)(z ? g.ihz : g.ihy);
#pragma unroll
    for (int e = 0; e < W; ++e) s[e] = hi ? (t[e] - xc[e]) * ih : (T)0;
  }
}

// chunks per thread per warp group of pass 1 (amortises the per-group setup)
constexpr int P1_U = 4;

// PU chunks (stride 32) of one (set, block) segment; KIND: 0 box, 1 distance
// block, 2 global set.  Reductions are summed in T per chunk, in fp64 across
// chunks, and reduced across the warp once per group.
template <class T, int KIND>
__device__ __forceinline__ void p1_seg(const Prob<T>& P, const Ctrl& C, int i, int bl, const IterFlags& f,
                                       int par, int cbase, int nch, int lane, const T* xs_rd, double* acc,
                                       int nv, unsigned* h1) {
  constexpr int W = VT<T>::W;
  const Geo& g = P.g;
  const SetD<T>& S = P.set[i];
  const int prim = S.prim[bl];
  const bool pointwise = KIND != 2;
  const T* yr = S.y[par] + (int64_t)bl * g.ld;
  const T* vr = S.v[par] + (int64_t)bl * g.ld;
  T* yw = S.y[par ^ 1] + (int64_t)bl * g.ld;
  T* vw = S.v[par ^ 1] + (int64_t)bl * g.ld;
  T* vhp = S.vh0 + (int64_t)bl * g.ld;
  T* wp = S.w ? S.w + (int64_t)bl * g.ld : nullptr;
  T* sp = S.s ? S.s + (int64_t)bl * g.ld : nullptr;
  const T* lop = S.lo_vec ? S.lo_vec + (int64_t)bl * g.ld : nullptr;
  const T* hip = S.hi_vec ? S.hi_vec + (int64_t)bl * g.ld : nullptr;
  const T rho = (T)C.rho[i], gam = (T)C.gamma[i], one = (T)1;
  const T irho = (T)(1.0 / C.rho[i]), i1rho = (T)(1.0 / (1.0 + C.rho[i]));
  const T tlo = (T)S.lo, thi = (T)S.hi;
  // fused round 1 of the radix search on w (fp32; see k_selectf): smem
  // histogram of the top 11 key bits, count + significand offset in 10-bit limbs
  unsigned* hc = (KIND == 2 && h1 && S.job >= 0) ? h1 + (S.job >> 1) * 3 * NBUCK : nullptr;
  const bool hsum = S.kind == K_L1;
  double d_w2 = 0, d_hv = 0, d_hh = 0, d_vh = 0, d_gv = 0, d_gg = 0, d_vv = 0, d_fn = 0, d_s2 = 0;
#pragma unroll 1
  for (int u = 0; u < P1_U; ++u) {
    const int c = cbase + u * 32 + lane;
    const bool valid = c < nch;
    const int pt0 = (valid ? c : nch - 1) * W;
    const Loc L = locate(g, pt0);
    T xc[W], yo[W], vo[W], lo[W], hi[W], mm[W], y0[W], v0[W], vh0[W], xo[W];
    VT<T>::ldT(P.x + pt0, xc);
    VT<T>::ldT(yr + pt0, yo);
    VT<T>::ldT(vr + pt0, vo);
    if (KIND == 0 && lop) VT<T>::ldT(lop + pt0, lo);
    if (KIND == 0 && hip) VT<T>::ldT(hip + pt0, hi);
    if (KIND == 1) VT<T>::ldT(P.m + pt0, mm);
    if (f.dots) {
      VT<T>::ldT(vhp + pt0, vh0);
      VT<T>::ldT(xs_rd + pt0, xo);
      if (pointwise) {
        VT<T>::ldT(yw + pt0, y0);
        VT<T>::ldT(vw + pt0, v0);
      }
    }
    T s[W], s0[W];
    prim_chunkT<T>(g, prim, P.x, pt0, lane, L, xc, s);
    if (f.dots) prim_chunkT<T>(g, prim, xs_rd, pt0, lane, L, xo, s0);
    T a_w2 = 0, a_hv = 0, a_hh = 0, a_vh = 0, a_gv = 0, a_gg = 0, a_vv = 0, a_fn = 0, a_s2 = 0;
    T yn[W], vn[W], wv[W], vh[W], st_s[W];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const bool pad = !valid || pad_vec(g, prim, L, e);
      const T sv = pad ? (T)0 : s[e];
      st_s[e] = sv;
      const T xbar = gam * sv + (one - gam) * yo[e];                   // relaxation
      // fp64 keeps the oracle's exact divisions; fp32 multiplies by reciprocals
      const T w = xbar - (sizeof(T) == 8 ? vo[e] / rho : vo[e] * irho);
      wv[e] = pad ? (T)0 : w;
      if (pointwise) {
        T y;
        if (KIND == 1) {
          y = sizeof(T) == 8 ? (mm[e] + rho * w) / (one + rho) : (mm[e] + rho * w) * i1rho;  // Eq. 22
        } else {
          const T l = lop ? lo[e] : tlo;
          const T h = hip ? hi[e] : thi;
          y = w < l ? l : (w > h ? h : w);                             // box clamp
          if (f.check && !pad) {
            const T cl = sv < l ? l : (sv > h ? h : sv);
            a_fn += (sv - cl) * (sv - cl);
          }
        }
        const T vt = rho * (y - w);                                    // Eq. 21 as rho (y - w), L26
        yn[e] = pad ? (T)0 : y;
        vn[e] = pad ? (T)0 : vt;
        if (f.dots && !pad) {
          const T dg = y0[e] - y;
          const T dv = vt - v0[e];
          a_gv += dg * dv; a_gg += dg * dg; a_vv += dv * dv;
        }
      } else if (!pad) {
        a_w2 += w * w;
      }
      if (f.adapt) {                                                   // Alg. 2 line 1
        const T vht = vo[e] + rho * (yo[e] - sv);
        vh[e] = pad ? (T)0 : vht;
        if (f.dots && !pad) {
          const T dvh = vht - vh0[e];
          const T dh = sv - s0[e];
          a_hv += dh * dvh; a_hh += dh * dh; a_vh += dvh * dvh;
        }
      }
      if (f.check && !pad) a_s2 += sv * sv;
    }
    if (valid) {
      if (pointwise) {
        VT<T>::stT(yw + pt0, yn);
        VT<T>::stT(vw + pt0, vn);
      } else {
        VT<T>::stT(wp + pt0, wv);
        if (f.check && sp) VT<T>::stT(sp + pt0, st_s);
      }
      if (f.adapt) VT<T>::stT(vhp + pt0, vh);
    }
    if (sizeof(T) == 4 && KIND == 2 && hc && valid) {
      int pd = -1;
      unsigned pc = 0, pa = 0, pb = 0;
#pragma unroll
      for (int e = 0; e < W; ++e) {
        if (pad_vec(g, prim, L, e)) continue;
        const unsigned key = __float_as_uint((float)wv[e]) & 0x7fffffffu;
        const int d = (int)(key >> 20);
        if (d != pd) {
          if (pd >= 0) {
            atomicAdd(&hc[pd], pc);
            if (hsum) { atomicAdd(&hc[NBUCK + pd], pa); atomicAdd(&hc[2 * NBUCK + pd], pb); }
          }
          pd = d; pc = 0; pa = 0; pb = 0;
        }
        pc += 1;
        pa += key & 1023u;
        pb += (key >> 10) & 1023u;
      }
      if (pd >= 0) {
        atomicAdd(&hc[pd], pc);
        if (hsum) { atomicAdd(&hc[NBUCK + pd], pa); atomicAdd(&hc[2 * NBUCK + pd], pb); }
      }
    }
    d_w2 += (double)a_w2; d_hv += (double)a_hv; d_hh += (double)a_hh; d_vh += (double)a_vh;
    d_gv += (double)a_gv; d_gg += (double)a_gg; d_vv += (double)a_vv; d_fn += (double)a_fn;
    d_s2 += (double)a_s2;
  }
  const int base = i * NSLOT;
  if (KIND == 2 && (S.kind == K_L2 || S.kind == K_ANN)) warp_acc(acc, nv, base + SLOT_W2, d_w2);
  if (f.dots) {
    warp_acc(acc, nv, base + SLOT_HV, d_hv);
    warp_acc(acc, nv, base + SLOT_HH, d_hh);
    warp_acc(acc, nv, base + SLOT_VHVH, d_vh);
    if (pointwise) {
      warp_acc(acc, nv, base + SLOT_GV, d_gv);
      warp_acc(acc, nv, base + SLOT_GG, d_gg);
      warp_acc(acc, nv, base + SLOT_VV, d_vv);
    }
  }
  if (f.check) {
    if (KIND == 0) warp_acc(acc, nv, base + SLOT_FN, d_fn);
    warp_acc(acc, nv, base + SLOT_S2, d_s2);
  }
}

// pass-1 finaliser (one CTA): Alg. 2 / Eq. 26-27 sums into the control
// block, l2 / annulus radial factors (Table 1, L7)
template <class T>
__device__ inline void fin_pass1(const Prob<T>& P, Ctrl& C, const double* stage) {
  const int nv = P.P * NSLOT + NEVOL;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    const double val = stage[v];
    if (v < P.P * NSLOT) C.sums[v / NSLOT][v % NSLOT] = val;
    else C.evol[v - P.P * NSLOT] = val;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < P.P; ++i) {
      const int kd = P.set[i].kind;
      if (kd != K_L2 && kd != K_ANN) continue;
      const double n = sqrt(stage[i * NSLOT + SLOT_W2]);
      double fct = 1.0;
      int z = 0;
      if (n == 0.0) z = (C.sig_lo[i] > 0.0);
      else if (n > C.sig_hi[i]) fct = C.sig_hi[i] / n;
      else if (n < C.sig_lo[i]) fct = C.sig_lo[i] / n;
      C.ann_scale[i] = fct;
      C.ann_zero[i] = z;
    }
  }
}

template <class T, int AD, int CK>
__global__ void __launch_bounds__(BLOCK, 2) k_pass1t(const __grid_constant__ Prob<T> P) {
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  extern __shared__ double acc[];
  __shared__ double sh[NWARP + 1];
  const Geo& g = P.g;
  const IterFlags f = iter_flags<AD, CK>(C);
  const int nv = P.P * NSLOT + NEVOL;
  const int par = C.k & 1;
  const int a = C.adapt_calls;
  const T* xs_rd = P.xs[(a + 1) & 1];
  T* xs_wr = P.xs[a & 1];
  const int hcount = C.hist_count, hhead = C.hist_head;
  const int hslot = (hhead + 1) % HIST_S;
  for (int v = threadIdx.x; v < NWARP * nv; v += BLOCK) acc[v] = 0.0;
  unsigned* h1 = P.fuse_r1 ? reinterpret_cast<unsigned*>(reinterpret_cast<char*>(acc) + P.h1_off) : nullptr;
  if (h1)
    for (int v = threadIdx.x; v < P.fuse_r1 * 3 * NBUCK; v += BLOCK) h1[v] = 0u;
  __syncthreads();
  const int nch = g.N / W;
  const int gch = 32 * P1_U;                           // chunks per warp group
  const int gps = (nch + gch - 1) / gch;               // warp groups per segment
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * NWARP;
  const int g0 = blockIdx.x * NWARP + (threadIdx.x >> 5);
  // chunk-major order: the segments of one chunk range are processed by
  // consecutive warps, so x (and x^{k0}) come from DRAM once
  const int nseg = P.nseg1;
  const int total = gps * nseg;
  for (int grp = g0; grp < total; grp += nw) {
    const int cg = grp / nseg;
    const int seg = grp - cg * nseg;
    const int cbase = cg * gch;
    if (seg == 0) {   // x history (Eq. 27) and Alg. 2's x snapshot
      double x2 = 0.0, d2[HIST_S] = {0, 0, 0, 0, 0};
      for (int u = 0; u < P1_U; ++u) {
        const int c = cbase + u * 32 + lane;
        const bool valid = c < nch;
        const int pt0 = (valid ? c : nch - 1) * W;
        T xc[W];
        VT<T>::ldT(P.x + pt0, xc);
        if (f.check) {
          T h[HIST_S][W];
#pragma unroll
          for (int js = 0; js < HIST_S; ++js)
            if ((hhead - js + HIST_S) % HIST_S < hcount) VT<T>::ldT(P.hist[js] + pt0, h[js]);
          T t2 = 0;
#pragma unroll
          for (int e = 0; e < W; ++e) t2 += valid ? xc[e] * xc[e] : (T)0;
          x2 += (double)t2;
#pragma unroll
          for (int js = 0; js < HIST_S; ++js) {
            if ((hhead - js + HIST_S) % HIST_S >= hcount) continue;
            T t = 0;
#pragma unroll
            for (int e = 0; e < W; ++e) {
              const T d = xc[e] - h[js][e];
              t += valid ? d * d : (T)0;
            }
            d2[js] += (double)t;
          }
        }
        if (valid) {
          VT<T>::stT(P.hist[hslot] + pt0, xc);
          if (f.adapt) {
            VT<T>::stT(xs_wr + pt0, xc);
            if (pt0 >= g.N - g.plane) {   // the upper ghost plane too (x^{k0} at z+1 on a z slab)
              T xg_[W];
              VT<T>::ldT(P.x + pt0 + g.plane, xg_);
              VT<T>::stT(xs_wr + pt0 + g.plane, xg_);
            }
          }
        }
      }
      if (f.check) {
        warp_acc(acc, nv, P.P * NSLOT, x2);
#pragma unroll
        for (int js = 0; js < HIST_S; ++js)
          if ((hhead - js + HIST_S) % HIST_S < hcount) warp_acc(acc, nv, P.P * NSLOT + 1 + js, d2[js]);
      }
    } else {
      const int i = P.seg_set[seg], bl = P.seg_blk[seg];
      switch (P.set[i].kind) {
        case K_BOUNDS: p1_seg<T, 0>(P, C, i, bl, f, par, cbase, nch, lane, xs_rd, acc, nv, h1); break;
        case K_DIST: p1_seg<T, 1>(P, C, i, bl, f, par, cbase, nch, lane, xs_rd, acc, nv, h1); break;
        default: p1_seg<T, 2>(P, C, i, bl, f, par, cbase, nch, lane, xs_rd, acc, nv, h1); break;
      }
    }
  }
  if (h1) {   // flush the round-1 histograms (exact integer sums) to global
    __syncthreads();
    for (int jj = 0; jj < P.fuse_r1; ++jj) {
      const int jb = 2 * jj;
      const unsigned* hc = h1 + jj * 3 * NBUCK;
      for (int d = threadIdx.x; d < NBUCK; d += BLOCK) {
        const unsigned cnt = hc[d];
        if (!cnt) continue;
        atomicAdd(P.gh_cnt + (size_t)jb * NBUCK + d, cnt);
        const unsigned long long base = ((d >> 3) ? (1ull << 23) : 0ull) + ((unsigned long long)(d & 7) << 20);
        const unsigned long long sum = (unsigned long long)cnt * base + hc[NBUCK + d] +
                                       ((unsigned long long)hc[2 * NBUCK + d] << 10);
        atomicAdd(P.gh_s0 + (size_t)jb * NBUCK + d, sum);
      }
    }
  }
  double* stage = P.partials + (size_t)gridDim.x * nv;
  if (finish_reduction(acc, nv, P.partials, P.counter, stage, sh)) {
    if (P.nranks > 1) {
      publish(P, stage, nv, threadIdx.x, BLOCK);
      return;
    }
    fin_pass1<T>(P, C, stage);
    if (h1) {   // resolve round 1 of the w jobs (k_selectf continues at round 2)
      __syncthreads();
      for (int jj = 0; jj < P.fuse_r1; ++jj) {
        const int jb = 2 * jj;
        Job& J = C.job[jb];
        if (J.mode == JM_SEARCH && J.round == 0) {
          resolve_round<T>(P, J, 1, P.gh_cnt + (size_t)jb * NBUCK, P.gh_s0 + (size_t)jb * NBUCK,
                           P.gh_s1 + (size_t)jb * NBUCK);
        }
        for (int d = threadIdx.x; d < NBUCK; d += BLOCK) {
          P.gh_cnt[(size_t)jb * NBUCK + d] = 0u;
          P.gh_s0[(size_t)jb * NBUCK + d] = 0ull;
          P.gh_s1[(size_t)jb * NBUCK + d] = 0ull;
        }
        __syncthreads();
      }
    }
  }
}

// ------------------------------------------------------------ pass 2
// KIND: 0 l1 ball (soft threshold at theta), 1 cardinality (keep > tau and the
// first keep_eq == tau in index order), 2 l2 ball / annulus (radial factor)
template <class T, int KIND>
__device__ __forceinline__ void p2_tile(const Prob<T>& P, const Ctrl& C, int i, int bl, int lt, int tpb,
                                        const IterFlags& f, int par, double* acc, int nv, int* s_w) {
  using K = KeyT<T>;
  using U = typename K::U;
  constexpr int W = VT<T>::W;
  const Geo& g = P.g;
  const SetD<T>& S = P.set[i];
  const int prim = S.prim[bl];
  const int nch = g.N / W;
  const int c = lt * BLOCK + threadIdx.x;
  const bool valid = c < nch;
  const int pt0 = (valid ? c : nch - 1) * W;
  const Loc L = locate(g, pt0);
  const int64_t off = (int64_t)bl * g.ld + pt0;
  T wv[W], y0[W], v0[W];
  VT<T>::ldT(S.w + off, wv);
  if (f.dots) {
    VT<T>::ldT(S.y[par ^ 1] + off, y0);
    VT<T>::ldT(S.v[par ^ 1] + off, v0);
  }
  bool pad[W];
#pragma unroll
  for (int e = 0; e < W; ++e) pad[e] = !valid || pad_vec(g, prim, L, e);
  T y[W];
  if (KIND == 0) {
    const Job& J = C.job[S.job];
    const T th = (T)J.theta;
    const bool done = J.mode == JM_DONE, keep = (J.mode == JM_INSIDE || J.mode == JM_ALL);
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const T w = wv[e];
      if (done) {
        const T a = (sizeof(T) == 8) ? (T)(fabs((double)w) - J.theta) : fabsf((float)w) - th;
        y[e] = a > (T)0 ? (w > (T)0 ? a : -a) : (T)0;   // soft threshold
      } else {
        y[e] = keep ? w : (T)0;
      }
    }
  } else if (KIND == 1) {
    const Job& J = C.job[S.job];
    const U tau = (U)J.tau;
    bool keep[W];
    int cnt = 0;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const U key = K::key(wv[e]);
      keep[e] = (J.mode == JM_ALL) || (J.mode == JM_DONE && key > tau);
      cnt += (J.mode == JM_DONE && !pad[e] && key == tau) ? 1 : 0;
    }
    if (J.mode == JM_DONE) {
      if (J.ties) {   // the first keep_eq entries == tau in index order (L6)
        const int* toff = P.tiecnt + (size_t)S.job * P.ntiles_max;
        long long r = (long long)toff[bl * tpb + lt] + block_excl_count(cnt, s_w);
#pragma unroll
        for (int e = 0; e < W; ++e)
          if (!pad[e] && K::key(wv[e]) == tau) { if (r < J.keep_eq) keep[e] = true; ++r; }
      } else {
#pragma unroll
        for (int e = 0; e < W; ++e) if (K::key(wv[e]) == tau) keep[e] = true;
      }
    }
#pragma unroll
    for (int e = 0; e < W; ++e) y[e] = keep[e] ? wv[e] : (T)0;
  } else {
    const T sc = (T)C.ann_scale[i];
    const int az = C.ann_zero[i];
#pragma unroll
    for (int e = 0; e < W; ++e)
      y[e] = az ? ((bl == 0 && pt0 + e == S.first_real) ? (T)C.sig_lo[i] : (T)0) : wv[e] * sc;
  }
  const T rho = (T)C.rho[i];
  T yn[W], vn[W];
  T a_gv = 0, a_gg = 0, a_vv = 0;
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const T yt = pad[e] ? (T)0 : y[e];
    const T vt = pad[e] ? (T)0 : rho * (yt - wv[e]);    // Eq. 21 as rho (y - w), L26
    yn[e] = yt;
    vn[e] = vt;
    if (f.dots && !pad[e]) {
      const T dg = y0[e] - yt;
      const T dv = vt - v0[e];
      a_gv += dg * dv; a_gg += dg * dg; a_vv += dv * dv;
    }
  }
  if (valid) {
    VT<T>::stT(S.y[par ^ 1] + off, yn);
    VT<T>::stT(S.v[par ^ 1] + off, vn);
  }
  if (f.dots) {
    warp_acc(acc, nv, i * 4 + 0, (double)a_gv);
    warp_acc(acc, nv, i * 4 + 1, (double)a_gg);
    warp_acc(acc, nv, i * 4 + 2, (double)a_vv);
  }
}

// pass-2 finaliser (one CTA): Alg. 2 beta-side sums and the Eq. 26
// numerators of the global sets
template <class T>
__device__ inline void fin_pass2(const Prob<T>& P, Ctrl& C, const double* stage) {
  const int nv = P.P * 4;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    const int i = v / 4, q = v % 4;
    if (!P.set[i].global) continue;
    const double val = stage[v];
    if (q == 0) C.sums[i][SLOT_GV] = val;
    if (q == 1) C.sums[i][SLOT_GG] = val;
    if (q == 2) C.sums[i][SLOT_VV] = val;
    if (q == 3 && P.set[i].sjob >= 0) C.sums[i][SLOT_FN] = val;
  }
}

template <class T, int AD, int CK>
__global__ void __launch_bounds__(BLOCK) k_pass2t(const __grid_constant__ Prob<T> P) {
  using K = KeyT<T>;
  using U = typename K::U;
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  extern __shared__ double acc[];
  __shared__ double sh[NWARP + 1];
  __shared__ int s_w[NWARP];
  const Geo& g = P.g;
  const IterFlags f = iter_flags<AD, CK>(C);
  const int nv = P.P * 4;
  const int par = C.k & 1;
  for (int v = threadIdx.x; v < NWARP * nv; v += BLOCK) acc[v] = 0.0;
  __syncthreads();
  const int nch = g.N / W;
  const int tpb = (nch + BLOCK - 1) / BLOCK;
  int sg = blockIdx.x / tpb, lt = blockIdx.x - sg * tpb;
  while (sg < P.nseg2) {
    const int i = P.seg2_set[sg], bl = P.seg2_blk[sg];
    switch (P.set[i].kind) {
      case K_L1: p2_tile<T, 0>(P, C, i, bl, lt, tpb, f, par, acc, nv, s_w); break;
      case K_CARD: p2_tile<T, 1>(P, C, i, bl, lt, tpb, f, par, acc, nv, s_w); break;
      default: p2_tile<T, 2>(P, C, i, bl, lt, tpb, f, par, acc, nv, s_w); break;
    }
    lt += gridDim.x;
    while (lt >= tpb) { lt -= tpb; ++sg; }
  }
  // Eq. 26 numerators of l1 / cardinality sets from s (check iterations)
  if (f.check) {
    for (int i = 0; i < P.P; ++i) {
      const SetD<T>& S = P.set[i];
      if (!S.global || S.sjob < 0) continue;
      const Job& Js = C.job[S.sjob];
      double fn = 0.0;
      if (Js.mode == JM_DONE) {
        const int tot = S.nblk * nch;
        for (int q = blockIdx.x * BLOCK + threadIdx.x; q < tot; q += gridDim.x * BLOCK) {
          const int bl = q / nch, c = q - bl * nch;
          T sv[W];
          VT<T>::ldT(S.s + (int64_t)bl * g.ld + (int64_t)c * W, sv);
          T a2 = 0;
#pragma unroll
          for (int e = 0; e < W; ++e) {
            if (S.kind == K_L1) {
              const T th = (T)Js.theta;
              const T a = sv[e] < (T)0 ? -sv[e] : sv[e];
              const T m = a < th ? a : th;
              a2 += m * m;
            } else if (K::key(sv[e]) < (U)Js.tau) {
              a2 += sv[e] * sv[e];
            }
          }
          fn += (double)a2;
        }
      }
      warp_acc(acc, nv, i * 4 + 3, fn);
    }
  }
  double* stage = P.partials + (size_t)gridDim.x * nv;
  if (finish_reduction(acc, nv, P.partials, P.counter, stage, sh)) {
    if (P.nranks > 1) publish(P, stage, nv, threadIdx.x, BLOCK);
    else fin_pass2<T>(P, C, stage);
  }
}

}  // namespace sip
