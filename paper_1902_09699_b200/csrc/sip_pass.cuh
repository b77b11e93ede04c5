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
#include "sip_stage.cuh"
#include "sip_select2.cuh"

#ifndef P2_H
#define P2_H 2        // pass 2: tiles per CTA step (one chunk of each per thread)
#endif
#ifndef P2_H0
#define P2_H0 4       // iterations without the Alg. 2 products (AD == 0): four (C5-L1 pass 2 11.45 -> 10.7 ms per step, C4 unchanged)
#endif
#ifndef P2_MINB
#define P2_MINB 4
#endif
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

// ------------------------------------------------------------ pass 1
// Segment-major over a contiguous chunk range per CTA.  A segment is the x
// work (history ring, Alg. 2 x snapshot, Eq. 27 sums) or one (set, block)
// pair; the CTA runs every segment over its range, one thread per chunk of
// W = 16 / sizeof(T) points, with the set kind, the primitive operator and
// the iteration type fixed at compile time (no per-element dispatch).  x and
// its neighbours are re-read per segment from L1 / L2 (x was just written by
// the CG); y_i, v_i and the outputs stream through DRAM once.  Per-thread
// fp64 accumulators are reduced once per (warp, segment) into the per-warp
// shared slots.

// A_prim x at the W points of a chunk in the storage precision (Eq. 8);
// pad entries come out 0
template <class T, int PRIM>
__device__ __forceinline__ void prim_chunk(const Geo& g, const T* x, int pt0, const T* xc, bool lastx, bool padc,
                                           T* s) {
  constexpr int W = VT<T>::W;
  if (PRIM == PRIM_I) {
#pragma unroll
    for (int e = 0; e < W; ++e) s[e] = xc[e];
  } else if (PRIM == PRIM_X) {
    const T xr = lastx ? (T)0 : x[pt0 + W];
    const T ih = (T)g.ihx;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const T nx_ = e < W - 1 ? xc[e + 1] : xr;
      s[e] = (lastx && e == W - 1) ? (T)0 : (nx_ - xc[e]) * ih;
    }
  } else {
    T t[W];
    VT<T>::ldT(x + pt0 + (PRIM == PRIM_Z ? g.plane : g.nx), t);
    const T ih = (T)(PRIM == PRIM_Z ? g.ihz : g.ihy);
#pragma unroll
    for (int e = 0; e < W; ++e) s[e] = padc ? (T)0 : (t[e] - xc[e]) * ih;
  }
}

// chunk location: whole-chunk pad (D_z: last global plane; D_y: last row)
// and whether the chunk holds the last point of its x row (D_x pad)
template <int PRIM>
__device__ __forceinline__ void chunk_pads(const Geo& g, int pt0, int W, bool* padc, bool* lastx) {
  const int iz = (int)g.dplane.div((uint32_t)pt0);
  const int r = pt0 - iz * g.plane;
  const int iy = (int)g.dnx.div((uint32_t)r);
  const int ix = r - iy * g.nx;
  *padc = PRIM == PRIM_Z ? (iz + g.z0 >= g.nz_g - 1) : PRIM == PRIM_Y ? (iy >= g.ny - 1) : false;
  *lastx = PRIM == PRIM_X && (ix + W >= g.nx);
}

// ------------------------------------------------------------ init (vectorised)
// k_initv: k_init for the vectorised path, one thread per chunk: x = m
// (unless warm), the history ring's first x, y_i = A_i m, v_i = 0 (reading
// L13), and the l1 / l2 norms of A_i m for the relative parameters (L4).
// Fiber sets' other parity, snapshots and w / s get zeros (the fiber kernels
// leave pads alone); SIP_POISON fills the fields the pass kernels write
// before reading with NaN.
template <class T>
__global__ void __launch_bounds__(BLOCK) k_initv(const __grid_constant__ Prob<T> P, int init_x, int init_yv) {
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  extern __shared__ double acc[];
  __shared__ double sh[NWARP + 1];
  const Geo& g = P.g;
  const int nv = P.P * 2;
  for (int v = threadIdx.x; v < NWARP * nv; v += BLOCK) acc[v] = 0.0;
  __syncthreads();
  const int nch = g.N / W;
  const T zero[W] = {};
  T nan_[W];
#pragma unroll
  for (int e = 0; e < W; ++e) nan_[e] = (T)NAN;
  double n1[MAXP], n2[MAXP];
  for (int i = 0; i < MAXP; ++i) { n1[i] = 0.0; n2[i] = 0.0; }
  for (int c = blockIdx.x * BLOCK + threadIdx.x; c < nch; c += gridDim.x * BLOCK) {
    const int pt0 = c * W;
    T mc[W];
    VT<T>::ldT(P.m + pt0, mc);
    if (init_x) VT<T>::stT(P.x + pt0, mc);
    T xc[W];
    if (init_x) {
#pragma unroll
      for (int e = 0; e < W; ++e) xc[e] = mc[e];
    } else {
      VT<T>::ldT(P.x + pt0, xc);
    }
    VT<T>::stT(P.hist[0] + pt0, xc);
    if (P.poison) { VT<T>::stT(P.xs[0] + pt0, nan_); VT<T>::stT(P.xs[1] + pt0, nan_); }
    for (int i = 0; i < P.P; ++i) {
      const SetD<T>& S = P.set[i];
      for (int bl = 0; bl < S.nblk; ++bl) {
        const int prim = S.prim[bl];
        bool padc = false, lastx = false;
        T sv[W];
        switch (prim) {
          case PRIM_Z: chunk_pads<PRIM_Z>(g, pt0, W, &padc, &lastx); prim_chunk<T, PRIM_Z>(g, P.m, pt0, mc, lastx, padc, sv); break;
          case PRIM_Y: chunk_pads<PRIM_Y>(g, pt0, W, &padc, &lastx); prim_chunk<T, PRIM_Y>(g, P.m, pt0, mc, lastx, padc, sv); break;
          case PRIM_X: chunk_pads<PRIM_X>(g, pt0, W, &padc, &lastx); prim_chunk<T, PRIM_X>(g, P.m, pt0, mc, lastx, padc, sv); break;
          default: prim_chunk<T, PRIM_I>(g, P.m, pt0, mc, false, false, sv); break;
        }
        T a1 = 0, a2 = 0;
#pragma unroll
        for (int e = 0; e < W; ++e) { a1 += sv[e] < (T)0 ? -sv[e] : sv[e]; a2 += sv[e] * sv[e]; }
        n1[i] += (double)a1;
        n2[i] += (double)a2;
        const int64_t off = (int64_t)bl * g.ld + pt0;
        if (init_yv) { VT<T>::stT(S.y[1] + off, sv); VT<T>::stT(S.v[1] + off, zero); }
        if (S.fib || P.poison) {
          const T* f = S.fib ? zero : nan_;
          VT<T>::stT(S.y[0] + off, f); VT<T>::stT(S.v[0] + off, f); VT<T>::stT(S.vh0 + off, f);
          if (S.w) VT<T>::stT(S.w + off, f);
          if (S.s) VT<T>::stT(S.s + off, f);
        }
      }
    }
  }
  for (int i = 0; i < P.P; ++i) {
    warp_acc(acc, nv, 2 * i, n1[i]);
    warp_acc(acc, nv, 2 * i + 1, n2[i]);
  }
  double* stage = P.partials + (size_t)gridDim.x * nv;
  if (finish_reduction(acc, nv, P.partials, P.counter, stage, sh)) {
    if (P.nranks > 1) publish(P, stage, nv, threadIdx.x, BLOCK);
    else if (threadIdx.x == 0) fin_init<T>(P, C, stage);
  }
}

// staged arrays of a pass-1 segment (Stage2 slots)
enum P1Arr { A_X = 0, A_XN, A_Y, A_V, A_M, A_HI, A_VH0, A_XS, A_XSN, A_Y0, A_V0, A_NP1 };
constexpr int P1_NA_PLAIN = 6;    // x, x+d, y, v, m or lo, hi
constexpr int P1_NA_ADAPT = A_NP1;

template <class T>
__device__ __forceinline__ void ld_s(const char* base, int idx, T* o) {   // chunk idx of a staged tile
  VT<T>::ldT_s(reinterpret_cast<const T*>(base) + idx * VT<T>::W, o);
}

// one (set, block) segment over chunks [c0, c1).  KIND: 0 box, 1 distance
// block (Eq. 22), 2 global set (w stored for pass 2)
template <class T, int KIND, int PRIM, int AD, int CK, int NA>
__device__ __forceinline__ void p1_run(const Prob<T>& P, const Ctrl& C, int i, int bl, const IterFlags& f,
                                       int par, int c0, int c1, const T* xs_rd, double* acc, int nv,
                                       Stage2<NA>& st, unsigned* ha) {
  constexpr int W = VT<T>::W;
  const Geo& g = P.g;
  const SetD<T>& S = P.set[i];
  const bool pointwise = KIND != 2;
  const bool adapt = AD == 2 ? f.adapt : AD == 1;
  const bool check = CK == 2 ? f.check : CK == 1;
  const bool dots = NA > A_VH0 && adapt && f.dots;
  const int64_t bo = (int64_t)bl * g.ld;
  const T* yr = S.y[par] + bo;
  const T* vr = S.v[par] + bo;
  T* yw = S.y[par ^ 1] + bo;
  T* vw = S.v[par ^ 1] + bo;
  T* vhp = S.vh0 + bo;
  T* wp = S.w ? S.w + bo : nullptr;
  T* sp = (check && S.s) ? S.s + bo : nullptr;
  const T* lop = S.lo_vec ? S.lo_vec + bo : nullptr;
  const T* hip = S.hi_vec ? S.hi_vec + bo : nullptr;
  const bool w2 = KIND == 2 && (S.kind == K_L2 || S.kind == K_ANN);
  const T rho = (T)C.rho[i], gam = (T)C.gamma[i], one = (T)1;
  const T irho = (T)(1.0 / C.rho[i]), i1rho = (T)(1.0 / (1.0 + C.rho[i]));
  const T tlo = (T)S.lo, thi = (T)S.hi;
  const int dn = PRIM == PRIM_Z ? g.plane : g.nx;   // neighbour offset of D_z / D_y
  const T ih = (T)(PRIM == PRIM_Z ? g.ihz : PRIM == PRIM_Y ? g.ihy : g.ihx);
  double d_w2 = 0, d_hv = 0, d_hh = 0, d_vh = 0, d_gv = 0, d_gg = 0, d_vv = 0, d_fn = 0, d_s2 = 0;
  double d_w1 = 0, d_s1 = 0;   // select v2: ||w||_1, ||s||_1 of an l1 radix job
  {   // the staged arrays of this segment (the issue below copies exactly these)
    constexpr bool nb = PRIM == PRIM_Z || PRIM == PRIM_Y;
    unsigned m = (1u << A_X) | (1u << A_Y) | (1u << A_V);
    if (nb) m |= 1u << A_XN;
    if (KIND == 1 || (KIND == 0 && lop)) m |= 1u << A_M;
    if (KIND == 0 && hip) m |= 1u << A_HI;
    if (NA > A_VH0 && dots) {
      m |= (1u << A_VH0) | (1u << A_XS);
      if (nb) m |= 1u << A_XSN;
      if (pointwise) m |= (1u << A_Y0) | (1u << A_V0);
    }
    st.set_layout(m);
  }
  const int ntile = (c1 - c0 + BLOCK - 1) / BLOCK;
  auto issue = [&](int t) {
    const int cs = c0 + t * BLOCK;
    const unsigned b = (unsigned)min(BLOCK, c1 - cs) * 16u;
    const unsigned bx = b + (PRIM == PRIM_X ? 16u : 0u);   // + the next chunk (x neighbour)
    const int64_t o = (int64_t)cs * W;
    const char* src[NA];
    unsigned by[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) { src[a] = nullptr; by[a] = 0; }
    src[A_X] = (const char*)(P.x + o); by[A_X] = bx;
    if (PRIM == PRIM_Z || PRIM == PRIM_Y) { src[A_XN] = (const char*)(P.x + o + dn); by[A_XN] = b; }
    src[A_Y] = (const char*)(yr + o); by[A_Y] = b;
    src[A_V] = (const char*)(vr + o); by[A_V] = b;
    if (KIND == 1) { src[A_M] = (const char*)(P.m + o); by[A_M] = b; }
    if (KIND == 0 && lop) { src[A_M] = (const char*)(lop + o); by[A_M] = b; }
    if (KIND == 0 && hip) { src[A_HI] = (const char*)(hip + o); by[A_HI] = b; }
    if (NA > A_VH0 && dots) {
      src[A_VH0] = (const char*)(vhp + o); by[A_VH0] = b;
      src[A_XS] = (const char*)(xs_rd + o); by[A_XS] = bx;
      if (PRIM == PRIM_Z || PRIM == PRIM_Y) { src[A_XSN] = (const char*)(xs_rd + o + dn); by[A_XSN] = b; }
      if (pointwise) {
        src[A_Y0] = (const char*)(yw + o); by[A_Y0] = b;
        src[A_V0] = (const char*)(vw + o); by[A_V0] = b;
      }
    }
    st.issue(t % st.ns, NA, src, by, P.p1_hint,
             (1u << A_X) | (1u << A_XN) | (NA > A_XS ? (1u << A_XS) : 0u) | (NA > A_XSN ? (1u << A_XSN) : 0u));
  };
  for (int q = 0; q < st.ns - 1 && q < ntile; ++q) issue(q);
  for (int t = 0; t < ntile; ++t) {
    if (t + st.ns - 1 < ntile) issue(t + st.ns - 1);
    const int s = t % st.ns;
    st.wait(s);
    const int c = c0 + t * BLOCK + (int)threadIdx.x;
    T hw_[W] = {}, hs_[W] = {};   // round-A keys of this chunk (zeros: not counted)
    if (c < c1) {
      const int pt0 = c * W;
      const int tid = threadIdx.x;
      bool padc, lastx;
      chunk_pads<PRIM>(g, pt0, W, &padc, &lastx);
      T xc[W], yo[W], vo[W];
      ld_s<T>(st.at(s, A_X), tid, xc);
      ld_s<T>(st.at(s, A_Y), tid, yo);
      ld_s<T>(st.at(s, A_V), tid, vo);
      // s = A x (Eq. 8), 0 on pads
      T sv_[W], s0_[W];
      auto prim_s = [&](int arr, int arrn, const T* c_, T* out) {
        if (PRIM == PRIM_I) {
#pragma unroll
          for (int e = 0; e < W; ++e) out[e] = c_[e];
        } else if (PRIM == PRIM_X) {
          const T xr = reinterpret_cast<const T*>(st.at(s, arr))[(tid + 1) * W];
#pragma unroll
          for (int e = 0; e < W; ++e) {
            const T nx_ = e < W - 1 ? c_[e + 1] : xr;
            out[e] = (lastx && e == W - 1) ? (T)0 : (nx_ - c_[e]) * ih;
          }
        } else {
          T tn[W];
          ld_s<T>(st.at(s, arrn), tid, tn);
#pragma unroll
          for (int e = 0; e < W; ++e) out[e] = padc ? (T)0 : (tn[e] - c_[e]) * ih;
        }
      };
      prim_s(A_X, A_XN, xc, sv_);
      T lo[W], hi[W], mm[W];
      if (KIND == 1) ld_s<T>(st.at(s, A_M), tid, mm);
      if (KIND == 0 && lop) ld_s<T>(st.at(s, A_M), tid, lo);
      if (KIND == 0 && hip) ld_s<T>(st.at(s, A_HI), tid, hi);
      T a_w2 = 0, a_hv = 0, a_hh = 0, a_vh = 0, a_gv = 0, a_gg = 0, a_vv = 0, a_fn = 0, a_s2 = 0;
      T yn[W], vn[W], wv[W], vh[W];
#pragma unroll
      for (int e = 0; e < W; ++e) {
        const bool pad = padc || (PRIM == PRIM_X && lastx && e == W - 1);
        const T sv = sv_[e];                                             // 0 on pads
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
            if (check && !pad) {
              const T cl = sv < l ? l : (sv > h ? h : sv);
              a_fn += (sv - cl) * (sv - cl);
            }
          }
          const T vt = rho * (y - w);                                    // Eq. 21 as rho (y - w), L26
          yn[e] = pad ? (T)0 : y;
          vn[e] = pad ? (T)0 : vt;
        } else if (w2 && !pad) {
          a_w2 += w * w;
        }
        if (adapt) vh[e] = pad ? (T)0 : vo[e] + rho * (yo[e] - sv);     // Alg. 2 line 1
        if (check && !pad) a_s2 += sv * sv;
      }
      if (dots) {   // Alg. 2 inner products against the k0 snapshots
        T xo[W], vh0[W];
        ld_s<T>(st.at(s, A_XS), tid, xo);
        ld_s<T>(st.at(s, A_VH0), tid, vh0);
        prim_s(A_XS, A_XSN, xo, s0_);
        T y0[W], v0[W];
        if (pointwise) {
          ld_s<T>(st.at(s, A_Y0), tid, y0);
          ld_s<T>(st.at(s, A_V0), tid, v0);
        }
#pragma unroll
        for (int e = 0; e < W; ++e) {
          const bool pad = padc || (PRIM == PRIM_X && lastx && e == W - 1);
          if (pad) continue;
          if (pointwise) {
            const T dg = y0[e] - yn[e];
            const T dv = vn[e] - v0[e];
            a_gv += dg * dv; a_gg += dg * dg; a_vv += dv * dv;
          }
          const T dvh = vh[e] - vh0[e];
          const T dh = sv_[e] - s0_[e];
          a_hv += dh * dvh; a_hh += dh * dh; a_vh += dvh * dvh;
        }
      }
      if (pointwise) {
        VT<T>::stT(yw + pt0, yn);
        VT<T>::stT(vw + pt0, vn);
      } else {
        VT<T>::stT(wp + pt0, wv);
        if (sp) VT<T>::stT(sp + pt0, sv_);
        if (KIND == 2 && ha) {   // select v2 round A: key counts of w (and s on checks)
#pragma unroll
          for (int e = 0; e < W; ++e) { hw_[e] = wv[e]; hs_[e] = sp ? sv_[e] : (T)0; }   // s is 0 on pads
          if (S.kind == K_L1) {                  // ||w||_1 (||s||_1) for the ball-inside test
            T t1 = 0, t2 = 0;
#pragma unroll
            for (int e = 0; e < W; ++e) {
              t1 += wv[e] < (T)0 ? -wv[e] : wv[e];
              if (sp) t2 += sv_[e] < (T)0 ? -sv_[e] : sv_[e];
            }
            d_w1 += (double)t1;
            d_s1 += (double)t2;
          }
        }
      }
      if (adapt) VT<T>::stT(vhp + pt0, vh);
      d_w2 += (double)a_w2; d_hv += (double)a_hv; d_hh += (double)a_hh; d_vh += (double)a_vh;
      d_gv += (double)a_gv; d_gg += (double)a_gg; d_vv += (double)a_vv; d_fn += (double)a_fn;
      d_s2 += (double)a_s2;
    }
    if (KIND == 2 && ha) {   // every lane of the warp (warp-grouped counts)
      // s counts on check iterations, else (l1) the sub-bucket sums of w
      hist_a<T>(ha, hw_, (P.sel_tsum && !check && S.kind == K_L1) ? ha + NBUCK : nullptr);
      if (sp) hist_a<T>(ha + NBUCK, hs_);
    }
    __syncthreads();   // stage s is refilled by the issue of tile t + ns
  }
  const int base = i * NSLOT;
  if (KIND == 2 && ha && S.kind == K_L1) {   // l1 sets use neither slot otherwise before pass 2
    warp_acc(acc, nv, base + SLOT_W2, d_w1);
    if (sp) warp_acc(acc, nv, base + SLOT_FN, d_s1);
  }
  if (w2) warp_acc(acc, nv, base + SLOT_W2, d_w2);
  if (dots) {
    warp_acc(acc, nv, base + SLOT_HV, d_hv);
    warp_acc(acc, nv, base + SLOT_HH, d_hh);
    warp_acc(acc, nv, base + SLOT_VHVH, d_vh);
    if (pointwise) {
      warp_acc(acc, nv, base + SLOT_GV, d_gv);
      warp_acc(acc, nv, base + SLOT_GG, d_gg);
      warp_acc(acc, nv, base + SLOT_VV, d_vv);
    }
  }
  if (check) {
    if (KIND == 0) warp_acc(acc, nv, base + SLOT_FN, d_fn);
    warp_acc(acc, nv, base + SLOT_S2, d_s2);
  }
}

// the x segment: history ring (Eq. 27), Alg. 2's x snapshot, ||x||^2 and
// ||x - x^{k-j}||^2 on check iterations
template <class T, int AD, int CK, int NA>
__device__ __forceinline__ void p1_xrun(const Prob<T>& P, const Ctrl& C, const IterFlags& f, int c0, int c1,
                                        T* xs_wr, double* acc, int nv, Stage2<NA>& st) {
  constexpr int W = VT<T>::W;
  const Geo& g = P.g;
  const bool adapt = AD == 2 ? f.adapt : AD == 1;
  const bool check = CK == 2 ? f.check : CK == 1;
  const int hcount = C.hist_count, hhead = C.hist_head;
  const int hslot = (hhead + 1) % HIST_S;
  double x2 = 0.0, d2[HIST_S] = {0, 0, 0, 0, 0};
  {
    unsigned m = 1u;
    if (check)
      for (int js = 0; js < HIST_S; ++js)
        if ((hhead - js + HIST_S) % HIST_S < hcount) m |= 1u << (1 + js);
    st.set_layout(m);
  }
  const int ntile = (c1 - c0 + BLOCK - 1) / BLOCK;
  auto issue = [&](int t) {
    const int cs = c0 + t * BLOCK;
    const unsigned b = (unsigned)min(BLOCK, c1 - cs) * 16u;
    const int64_t o = (int64_t)cs * W;
    const char* src[NA];
    unsigned by[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) { src[a] = nullptr; by[a] = 0; }
    src[0] = (const char*)(P.x + o); by[0] = b;
    if (check)
#pragma unroll
      for (int js = 0; js < HIST_S; ++js)
        if ((hhead - js + HIST_S) % HIST_S < hcount) { src[1 + js] = (const char*)(P.hist[js] + o); by[1 + js] = b; }
    st.issue(t % st.ns, NA, src, by, P.p1_hint, 1u);   // x: read again by every segment
  };
  for (int q = 0; q < st.ns - 1 && q < ntile; ++q) issue(q);
  for (int t = 0; t < ntile; ++t) {
    if (t + st.ns - 1 < ntile) issue(t + st.ns - 1);
    const int s = t % st.ns;
    st.wait(s);
    const int c = c0 + t * BLOCK + (int)threadIdx.x;
    if (c < c1) {
      const int pt0 = c * W;
      T xc[W];
      ld_s<T>(st.at(s, 0), threadIdx.x, xc);
      if (check) {
        T t2 = 0;
#pragma unroll
        for (int e = 0; e < W; ++e) t2 += xc[e] * xc[e];
        x2 += (double)t2;
#pragma unroll
        for (int js = 0; js < HIST_S; ++js) {
          if ((hhead - js + HIST_S) % HIST_S >= hcount) continue;
          T h[W];
          ld_s<T>(st.at(s, 1 + js), threadIdx.x, h);
          T tt = 0;
#pragma unroll
          for (int e = 0; e < W; ++e) {
            const T d = xc[e] - h[e];
            tt += d * d;
          }
          d2[js] += (double)tt;
        }
      }
      VT<T>::stT(P.hist[hslot] + pt0, xc);
      if (adapt) {
        VT<T>::stT(xs_wr + pt0, xc);
        if (pt0 >= g.N - g.plane) {   // the upper ghost plane too (x^{k0} at z+1 on a z slab)
          T xg_[W];
          VT<T>::ldT(P.x + pt0 + g.plane, xg_);
          VT<T>::stT(xs_wr + pt0 + g.plane, xg_);
        }
      }
    }
    __syncthreads();
  }
  if (check) {
    warp_acc(acc, nv, P.P * NSLOT, x2);
#pragma unroll
    for (int js = 0; js < HIST_S; ++js)
      if ((hhead - js + HIST_S) % HIST_S < hcount) warp_acc(acc, nv, P.P * NSLOT + 1 + js, d2[js]);
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

// k_pass1t: s = A x, relaxation, w, pointwise projections + duals, Alg. 2
// and Eq. 26/27 statistics (Algorithm 1 lines of P:279-288; Alg. 2 line 1)
template <class T, int AD, int CK>
__global__ void __launch_bounds__(BLOCK, AD == 0 ? 3 : 2) k_pass1t(const __grid_constant__ Prob<T> P) {
  pdl_begin();
  constexpr int W = VT<T>::W;
  constexpr int NA = AD == 0 ? P1_NA_PLAIN : P1_NA_ADAPT;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  extern __shared__ __align__(16) double acc[];
  __shared__ double sh[NWARP + 1];
  __shared__ uint64_t bars[SMAX];
  const Geo& g = P.g;
  const IterFlags f = iter_flags<AD, CK>(C);
  const int nv = P.P * NSLOT + NEVOL;
  const int par = C.k & 1;
  const int a = C.adapt_calls;
  const T* xs_rd = P.xs[(a + 1) & 1];
  T* xs_wr = P.xs[a & 1];
  for (int v = threadIdx.x; v < NWARP * nv; v += BLOCK) acc[v] = 0.0;
  Stage2<NA> st;
  const size_t accb = (((size_t)NWARP * nv * sizeof(double) + 127) / 128) * 128;
  const int pool = AD == 0 ? P.p1_pool : P.p1a_pool;
  st.init(bars, reinterpret_cast<char*>(acc) + accb, BLOCK, pool);
  // select v2 round A: two count histograms (w, s) after the stage pool
  unsigned* ha = P.selv2 ? reinterpret_cast<unsigned*>(reinterpret_cast<char*>(acc) + accb +
                                                       (size_t)pool * (BLOCK + 1) * 16)
                         : nullptr;
  if (ha)
    for (int d = threadIdx.x; d < 2 * NBUCK; d += BLOCK) ha[d] = 0u;
  const int nch = g.N / W;
  const int per = (nch + (int)gridDim.x - 1) / (int)gridDim.x;
  const int c0 = min(nch, (int)blockIdx.x * per), c1 = min(nch, c0 + per);
  // The CTA's range in sub-ranges of p1_sub chunks, every segment over one
  // sub-range before the next: x (and its z / y neighbour planes), which each
  // segment re-reads, is then still in L2 when the next segment asks for it.
  // The round-A counts of a set accumulate in shared memory across the
  // sub-ranges and are flushed when another set's counts need the buffer.
  const int sub = P.p1_sub > 0 ? P.p1_sub : max(per, 1);
  int hset = -1;                      // the set whose counts ha holds
  auto flush = [&]() {
    if (hset < 0) return;
    const SetD<T>& S = P.set[hset];
    hist_a_flush(ha, P.gh_cnt + (size_t)S.job * NBUCK);
    if (f.check && S.s) hist_a_flush(ha + NBUCK, P.gh_cnt + (size_t)S.sjob * NBUCK);
    else if (P.sel_tsum && !f.check && S.kind == K_L1) hist_a_flush(ha + NBUCK, P.gh_ta + (size_t)S.job * NBUCK);
    hset = -1;
  };
  for (int s0 = c0; s0 < c1; s0 += sub) {
    const int s1 = min(c1, s0 + sub);
    p1_xrun<T, AD, CK, NA>(P, C, f, s0, s1, xs_wr, acc, nv, st);
    for (int seg = 1; seg < P.nseg1; ++seg) {
      const int i = P.seg_set[seg], bl = P.seg_blk[seg];
      const int kd = P.set[i].kind;
      const int K = kd == K_BOUNDS ? 0 : (kd == K_DIST ? 1 : 2);
      unsigned* hai = (ha && K == 2 && P.set[i].job >= 0 && C.job[P.set[i].job].mode == JM_SEARCH) ? ha : nullptr;
      if (hai && hset != i) { flush(); hset = i; }
      switch (K * 4 + P.set[i].prim[bl]) {
#define P1CASE(KK, PP) \
        case KK * 4 + PP: p1_run<T, KK, PP, AD, CK, NA>(P, C, i, bl, f, par, s0, s1, xs_rd, acc, nv, st, hai); break;
        P1CASE(0, PRIM_I) P1CASE(0, PRIM_Z) P1CASE(0, PRIM_Y) P1CASE(0, PRIM_X)
        P1CASE(1, PRIM_I)
        P1CASE(2, PRIM_I) P1CASE(2, PRIM_Z) P1CASE(2, PRIM_Y) P1CASE(2, PRIM_X)
#undef P1CASE
        default: break;   // the distance block is I; blur/mask sets take the scalar kernels
      }
    }
  }
  if (ha) flush();
  double* stage = P.partials + (size_t)gridDim.x * nv;
  if (finish_reduction(acc, nv, P.partials, P.counter, stage, sh)) {
    if (P.nranks > 1) {
      publish(P, stage, nv, threadIdx.x, BLOCK);
      return;
    }
    fin_pass1<T>(P, C, stage);
  }
}

// dynamic shared memory of k_pass1t<T, AD, .>: per-warp slots + two stages
__host__ inline size_t pass1_smem(int P, int pool, bool selv2 = false) {
  const size_t accb = ((size_t)NWARP * (P * NSLOT + NEVOL) * sizeof(double) + 127) / 128 * 128;
  return accb + (size_t)pool * (BLOCK + 1) * 16 +
         (selv2 ? (size_t)2 * NBUCK * sizeof(unsigned) : 0);
}

// ------------------------------------------------------------ pass 2
// KIND: 0 l1 ball (soft threshold at theta), 1 cardinality (keep > tau and the
// first keep_eq == tau in index order), 2 l2 ball / annulus (radial factor)
template <class T, int KIND, int H>
__device__ __forceinline__ void p2_tile(const Prob<T>& P, const Ctrl& C, int i, int bl, int lp, int tpb,
                                        const IterFlags& f, int par, double* acc, int nv, int* s_w) {
  // tiles 2 lp and 2 lp + 1 of the block (BLOCK chunks each, k_tiecountf's
  // tiles): one chunk of each per thread, both chunks' loads in flight
  // together (one chunk per thread left too few bytes in flight)
  using K = KeyT<T>;
  using U = typename K::U;
  constexpr int W = VT<T>::W;
  const Geo& g = P.g;
  const SetD<T>& S = P.set[i];
  const int nch = g.N / W;
  const int prim = S.prim[bl];
  bool valid[H], pad[H][W];
  int pt0[H];
  int64_t off[H];
  T wv[H][W], y0[H][W], v0[H][W];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    const int c = (H * lp + h) * BLOCK + threadIdx.x;
    valid[h] = c < nch;
    pt0[h] = (valid[h] ? c : nch - 1) * W;
    off[h] = (int64_t)bl * g.ld + pt0[h];
    VT<T>::ldT(S.w + off[h], wv[h]);
    if (f.dots) {
      VT<T>::ldT(S.y[par ^ 1] + off[h], y0[h]);
      VT<T>::ldT(S.v[par ^ 1] + off[h], v0[h]);
    }
  }
#pragma unroll
  for (int h = 0; h < H; ++h) {   // pads once per chunk (no per-element operator dispatch)
    const int iz = (int)g.dplane.div((uint32_t)pt0[h]);
    const int r = pt0[h] - iz * g.plane;
    const int iy = (int)g.dnx.div((uint32_t)r);
    const bool padc = prim == PRIM_Z ? (iz + g.z0 >= g.nz_g - 1) : (prim == PRIM_Y ? iy >= g.ny - 1 : false);
    const bool lastx = prim == PRIM_X && (r - iy * g.nx + W >= g.nx);
#pragma unroll
    for (int e = 0; e < W; ++e) pad[h][e] = !valid[h] || padc || (lastx && e == W - 1);
  }
  T y[H][W];
  if (KIND == 0) {
    const Job& J = C.job[S.job];
    const T th = (T)J.theta;
    const bool done = J.mode == JM_DONE, keep = (J.mode == JM_INSIDE || J.mode == JM_ALL);
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int e = 0; e < W; ++e) {
        const T w = wv[h][e];
        if (done) {
          const T a = (sizeof(T) == 8) ? (T)(fabs((double)w) - J.theta) : fabsf((float)w) - th;
          y[h][e] = a > (T)0 ? (w > (T)0 ? a : -a) : (T)0;   // soft threshold
        } else {
          y[h][e] = keep ? w : (T)0;
        }
      }
  } else if (KIND == 1) {
    const Job& J = C.job[S.job];
    const U tau = (U)J.tau;
    bool keep[H][W];
    int cnt[H] = {};
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int e = 0; e < W; ++e) {
        const U key = K::key(wv[h][e]);
        keep[h][e] = (J.mode == JM_ALL) || (J.mode == JM_DONE && key > tau);
        cnt[h] += (J.mode == JM_DONE && !pad[h][e] && key == tau) ? 1 : 0;
      }
    if (J.mode == JM_DONE) {
      if (J.ties) {   // the first keep_eq entries == tau in index order (L6)
        const int* toff = P.tiecnt + (size_t)S.job * P.ntiles_max;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const int t = H * lp + h;
          const int ex = block_excl_count(cnt[h], s_w);   // every thread (block barrier inside)
          if (t >= tpb) continue;
          long long r = (long long)toff[bl * tpb + t] + ex;
#pragma unroll
          for (int e = 0; e < W; ++e)
            if (!pad[h][e] && K::key(wv[h][e]) == tau) { if (r < J.keep_eq) keep[h][e] = true; ++r; }
        }
      } else {
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
          for (int e = 0; e < W; ++e) if (K::key(wv[h][e]) == tau) keep[h][e] = true;
      }
    }
    unsigned long long hsum = 0;   // support fingerprint (test instrument)
#pragma unroll
    for (int h = 0; h < H; ++h) {
#pragma unroll
      for (int e = 0; e < W; ++e) y[h][e] = keep[h][e] ? wv[h][e] : (T)0;
      const unsigned long long gbase = (unsigned long long)bl * ((unsigned long long)g.nz_g * g.plane) +
                                       (unsigned long long)g.z0 * g.plane + (unsigned long long)pt0[h];
#pragma unroll
      for (int e = 0; e < W; ++e)
        if (!pad[h][e] && y[h][e] != (T)0) hsum += supp_mix(gbase + e);
    }
    supp_add_warp(C, i, hsum);
  } else {
    const T sc = (T)C.ann_scale[i];
    const int az = C.ann_zero[i];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int e = 0; e < W; ++e)
        y[h][e] = az ? ((bl == 0 && pt0[h] + e == S.first_real) ? (T)C.sig_lo[i] : (T)0) : wv[h][e] * sc;
  }
  const T rho = (T)C.rho[i];
  T a_gv = 0, a_gg = 0, a_vv = 0;
#pragma unroll
  for (int h = 0; h < H; ++h) {
    T yn[W], vn[W];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const T yt = pad[h][e] ? (T)0 : y[h][e];
      const T vt = pad[h][e] ? (T)0 : rho * (yt - wv[h][e]);    // Eq. 21 as rho (y - w), L26
      yn[e] = yt;
      vn[e] = vt;
      if (f.dots && !pad[h][e]) {
        const T dg = y0[h][e] - yt;
        const T dv = vt - v0[h][e];
        a_gv += dg * dv; a_gg += dg * dg; a_vv += dv * dv;
      }
    }
    if (valid[h]) {
      VT<T>::stT(S.y[par ^ 1] + off[h], yn);
      VT<T>::stT(S.v[par ^ 1] + off[h], vn);
    }
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
    if (q == 3 && (P.set[i].sjob >= 0 || P.set[i].fib)) C.sums[i][SLOT_FN] = val;
  }
}

template <class T, int AD, int CK>
__global__ void __launch_bounds__(BLOCK, AD == 0 ? P2_MINB : 3) k_pass2t(const __grid_constant__ Prob<T> P) {
  pdl_begin();
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
  const int tpb = (nch + BLOCK - 1) / BLOCK;   // k_tiecountf's tiles per block
  constexpr int H = AD == 0 ? P2_H0 : P2_H;
  const int ppb = (tpb + H - 1) / H;           // tile groups per block
  int sg = blockIdx.x / ppb, lp = blockIdx.x - sg * ppb;
  while (sg < P.nseg2) {
    const int i = P.seg2_set[sg], bl = P.seg2_blk[sg];
    switch (P.set[i].kind) {
      case K_L1: p2_tile<T, 0, H>(P, C, i, bl, lp, tpb, f, par, acc, nv, s_w); break;
      case K_CARD: p2_tile<T, 1, H>(P, C, i, bl, lp, tpb, f, par, acc, nv, s_w); break;
      default: p2_tile<T, 2, H>(P, C, i, bl, lp, tpb, f, par, acc, nv, s_w); break;
    }
    lp += gridDim.x;
    while (lp >= ppb) { lp -= ppb; ++sg; }
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
          const int bl = (q >= nch) + (q >= 2 * nch), c = q - bl * nch;   // nblk <= 3
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
    if (P.nranks > 1) {
      __syncthreads();
      if (P.fibv)   // per-fiber sets: this rank's sums from the fiber kernels (run before pass 2)
        for (int v = threadIdx.x; v < nv; v += BLOCK)
          if (P.set[v / 4].fib) stage[v] += P.fibv[v];
      __syncthreads();
      publish(P, stage, nv, threadIdx.x, BLOCK);
    } else {
      fin_pass2<T>(P, C, stage);
    }
  }
}

}  // namespace sip
