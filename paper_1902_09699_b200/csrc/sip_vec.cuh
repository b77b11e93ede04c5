// sip_vec.cuh -- vectorised stencil kernels for the CG hot loop (sm_100a).
//
// Each thread owns W = 16 / sizeof(T) consecutive x points ("chunk": one
// 128-bit load per array).  Chunks of a warp are consecutive, so the x
// neighbours come from the adjacent lanes by shuffle (lanes 0 / 31 load their
// outer neighbour); the y and z neighbours are 128-bit loads of the adjacent
// rows / planes, issued unconditionally (the ghost planes of every N-field
// make the out-of-domain addresses valid) and masked afterwards.  Requires
// nx % W == 0; the scalar kernels of sip_kernels.cuh cover the general case.
#pragma once
#include "sip_kernels.cuh"

namespace sip {

template <class T> struct VT;
template <> struct VT<float> {
  using v = float4;
  static constexpr int W = 4;
  __device__ static void ld(const float* p, double* o) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  }
  __device__ static void st(float* p, const double* o) {
    *reinterpret_cast<float4*>(p) = make_float4((float)o[0], (float)o[1], (float)o[2], (float)o[3]);
  }
  __device__ static void ldcs(const float* p, double* o) {   // streaming (read once)
    float4 a = __ldcs(reinterpret_cast<const float4*>(p));
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  }
  __device__ static void ldT(const float* p, float* o) {     // native precision
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  }
  __device__ static void stT(float* p, const float* o) {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
  }
};
template <> struct VT<double> {
  using v = double2;
  static constexpr int W = 2;
  __device__ static void ld(const double* p, double* o) {
    double2 a = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = a.x; o[1] = a.y;
  }
  __device__ static void st(double* p, const double* o) {
    *reinterpret_cast<double2*>(p) = make_double2(o[0], o[1]);
  }
  __device__ static void ldcs(const double* p, double* o) {
    double2 a = __ldcs(reinterpret_cast<const double2*>(p));
    o[0] = a.x; o[1] = a.y;
  }
  __device__ static void ldT(const double* p, double* o) { ld(p, o); }
  __device__ static void stT(double* p, const double* o) { st(p, o); }
};

// the 7-point neighbourhood of a chunk (values already in the fetched form)
template <int W>
struct Nbr {
  double c[W], zm[W], zp[W], ym[W], yp[W];
  double xl, xr;
};

// fetch p (USE_P: p_new = T(r + beta p_old), else r or a plain vector)
template <class T, bool USE_P>
__device__ __forceinline__ void fetch5(const Geo& g, const T* r, const T* p, double beta, int pt0,
                                       bool has_y, Nbr<VT<T>::W>& n) {
  constexpr int W = VT<T>::W;
  double a[5][W], b[5][W];
  const int off[5] = {0, -g.plane, g.plane, -g.nx, g.nx};
  const int np = has_y ? 5 : 3;
#pragma unroll
  for (int q = 0; q < 5; ++q)
    if (q < np) VT<T>::ld(r + pt0 + off[q], a[q]);
  if (USE_P) {
#pragma unroll
    for (int q = 0; q < 5; ++q)
      if (q < np) VT<T>::ld(p + pt0 + off[q], b[q]);
  }
#pragma unroll
  for (int e = 0; e < W; ++e) {
    auto f = [&](int q) { return USE_P ? (double)(T)(a[q][e] + beta * b[q][e]) : a[q][e]; };
    n.c[e] = f(0);
    n.zm[e] = f(1);
    n.zp[e] = f(2);
    n.ym[e] = has_y ? f(3) : 0.0;
    n.yp[e] = has_y ? f(4) : 0.0;
  }
}

// x neighbours by shuffle; warp-edge lanes load theirs
template <class T, bool USE_P>
__device__ __forceinline__ void fetch_x(const T* r, const T* p, double beta, int pt0, int lane,
                                        Nbr<VT<T>::W>& n) {
  constexpr int W = VT<T>::W;
  n.xl = __shfl_up_sync(0xffffffffu, n.c[W - 1], 1);
  n.xr = __shfl_down_sync(0xffffffffu, n.c[0], 1);
  if (lane == 0) {
    n.xl = USE_P ? (double)(T)((double)r[pt0 - 1] + beta * (double)p[pt0 - 1]) : (double)r[pt0 - 1];
  }
  if (lane == 31) {
    n.xr = USE_P ? (double)(T)((double)r[pt0 + W] + beta * (double)p[pt0 + W]) : (double)r[pt0 + W];
  }
}

// (C p) at the W points of the chunk (same arithmetic as apply_C_at)
template <int W>
__device__ __forceinline__ void apply_C_vec(const Ctrl& C, const Geo& g, bool has_z, bool has_y, bool has_x,
                                            const Nbr<W>& n, int ix0, int iy, int gz, double* q) {
  const bool zlo = gz >= 1, zhi = gz < g.nz_g - 1;
  const bool ylo = iy >= 1, yhi = iy < g.ny - 1;
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const double p0 = n.c[e];
    double v = C.cI * p0;
    if (has_z) {
      double a = 0.0;
      if (zlo) a += p0 - n.zm[e];
      if (zhi) a -= n.zp[e] - p0;
      v += C.cz * a;
    }
    if (has_y) {
      double a = 0.0;
      if (ylo) a += p0 - n.ym[e];
      if (yhi) a -= n.yp[e] - p0;
      v += C.cy * a;
    }
    if (has_x) {
      const int ix = ix0 + e;
      const double left = e > 0 ? n.c[e - 1] : n.xl;
      const double right = e < W - 1 ? n.c[e + 1] : n.xr;
      double a = 0.0;
      if (ix >= 1) a += p0 - left;
      if (ix < g.nx - 1) a -= right - p0;
      v += C.cx * a;
    }
    q[e] = v;
  }
}

// k_cg1v(j): p_j = r + beta p_{j-1}; <p_j, C p_j>
template <class T>
__global__ void __launch_bounds__(BLOCK) k_cg1v(const __grid_constant__ Prob<T> P, int j) {
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  const Geo& g = P.g;
  const int nch = g.N / W;
  if (j == 0 && C.zero_x) {
    for (int c = blockIdx.x * BLOCK + threadIdx.x; c < nch; c += gridDim.x * BLOCK) {
      double z[W] = {};
      VT<T>::st(P.x + c * W, z);
    }
    return;
  }
  if (!C.cg_active) return;
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  const double beta = C.beta;
  const T* pold = P.pb[(j + 1) & 1];
  T* pw = P.pb[j & 1];
  const bool hz = P.has[PRIM_Z], hy = P.has[PRIM_Y], hx = P.has[PRIM_X];
  const int lane = threadIdx.x & 31;
  double pq = 0.0;
  // uniform trip count per warp so every lane joins the shuffles
  const int stride = gridDim.x * BLOCK;
  for (int c0 = blockIdx.x * BLOCK + (threadIdx.x & ~31); c0 < nch; c0 += stride) {
    const int c = c0 + lane;
    const bool valid = c < nch;
    const int cc = valid ? c : nch - 1;
    const int pt0 = cc * W;
    Loc L = locate(g, pt0);
    Nbr<W> n;
    if (j > 0) fetch5<T, true>(g, P.r, pold, beta, pt0, hy, n);
    else fetch5<T, false>(g, P.r, pold, beta, pt0, hy, n);
    if (j > 0) fetch_x<T, true>(P.r, pold, beta, pt0, lane, n);
    else fetch_x<T, false>(P.r, pold, beta, pt0, lane, n);
    double q[W];
    apply_C_vec<W>(C, g, hz, hy, hx, n, L.ix, L.iy, L.gz, q);
    if (valid) {
      VT<T>::st(pw + pt0, n.c);
#pragma unroll
      for (int e = 0; e < W; ++e) pq += n.c[e] * q[e];
    }
  }
  pq = block_sum(pq, sh);
  if (threadIdx.x == 0) P.partials[blockIdx.x] = pq;
  if (last_block(P.counter)) {
    reduce_partials(P.partials, 1, out, sh);
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      if (out[0] > 0.0) {
        C.alpha = C.rr / out[0];
      } else {
        C.cg_active = 0;
        C.breakdown = 1;
      }
    }
  }
}

// k_cg2v(j): x += alpha p, r -= alpha C p; <r, r>
template <class T>
__global__ void __launch_bounds__(BLOCK) k_cg2v(const __grid_constant__ Prob<T> P, int j) {
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped || !C.cg_active) return;
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  const Geo& g = P.g;
  const int nch = g.N / W;
  const T* pv = P.pb[j & 1];
  const double alpha = C.alpha;
  const bool hz = P.has[PRIM_Z], hy = P.has[PRIM_Y], hx = P.has[PRIM_X];
  const int lane = threadIdx.x & 31;
  double rr = 0.0;
  const int stride = gridDim.x * BLOCK;
  for (int c0 = blockIdx.x * BLOCK + (threadIdx.x & ~31); c0 < nch; c0 += stride) {
    const int c = c0 + lane;
    const bool valid = c < nch;
    const int cc = valid ? c : nch - 1;
    const int pt0 = cc * W;
    Loc L = locate(g, pt0);
    Nbr<W> n;
    fetch5<T, false>(g, pv, nullptr, 0.0, pt0, hy, n);
    fetch_x<T, false>(pv, nullptr, 0.0, pt0, lane, n);
    double xv[W], rv[W];
    VT<T>::ldcs(P.x + pt0, xv);
    VT<T>::ldcs(P.r + pt0, rv);
    double q[W];
    apply_C_vec<W>(C, g, hz, hy, hx, n, L.ix, L.iy, L.gz, q);
#pragma unroll
    for (int e = 0; e < W; ++e) {
      xv[e] = xv[e] + alpha * n.c[e];
      rv[e] = (double)(T)(rv[e] - alpha * q[e]);
    }
    if (valid) {
      VT<T>::st(P.x + pt0, xv);
      VT<T>::st(P.r + pt0, rv);
#pragma unroll
      for (int e = 0; e < W; ++e) rr += rv[e] * rv[e];
    }
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

}  // namespace sip

namespace sip {

// forward differences of x at the W points of a chunk (Eq. 8; pads -> 0)
template <class T>
struct SChunk {
  static constexpr int W = VT<T>::W;
  double I[W], Z[W], Y[W], X[W];
  __device__ __forceinline__ double get(int prim, int e) const {
    switch (prim) {
      case PRIM_Z: return Z[e];
      case PRIM_Y: return Y[e];
      case PRIM_X: return X[e];
      default: return I[e];
    }
  }
};

template <class T>
__device__ __forceinline__ void s_chunk(const Prob<T>& P, const T* x, int pt0, int lane, const Loc& L,
                                        SChunk<T>& s) {
  constexpr int W = VT<T>::W;
  const Geo& g = P.g;
  VT<T>::ld(x + pt0, s.I);
  if (P.has[PRIM_Z]) {
    double t[W];
    VT<T>::ld(x + pt0 + g.plane, t);
    const bool zhi = L.gz < g.nz_g - 1;
#pragma unroll
    for (int e = 0; e < W; ++e) s.Z[e] = zhi ? (t[e] - s.I[e]) * g.ihz : 0.0;
  }
  if (P.has[PRIM_Y]) {
    double t[W];
    VT<T>::ld(x + pt0 + g.nx, t);
    const bool yhi = L.iy < g.ny - 1;
#pragma unroll
    for (int e = 0; e < W; ++e) s.Y[e] = yhi ? (t[e] - s.I[e]) * g.ihy : 0.0;
  }
  if (P.has[PRIM_X]) {
    double xr = __shfl_down_sync(0xffffffffu, s.I[0], 1);
    if (lane == 31) xr = (double)x[pt0 + W];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const double nx_ = e < W - 1 ? s.I[e + 1] : xr;
      s.X[e] = (L.ix + e < g.nx - 1) ? (nx_ - s.I[e]) * g.ihx : 0.0;
    }
  }
}

__device__ __forceinline__ bool pad_vec(const Geo& g, int prim, const Loc& L, int e) {
  switch (prim) {
    case PRIM_Z: return L.gz >= g.nz_g - 1;
    case PRIM_Y: return L.iy >= g.ny - 1;
    case PRIM_X: return L.ix + e >= g.nx - 1;
    default: return false;
  }
}

// vectorised k_pass1 (identical arithmetic; no blur operator)
template <class T>
__global__ void __launch_bounds__(BLOCK) k_pass1v(const __grid_constant__ Prob<T> P) {
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
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * BLOCK;
  for (int c0 = blockIdx.x * BLOCK + (threadIdx.x & ~31); c0 < nch; c0 += stride) {
    const int c = c0 + lane;
    const bool valid = c < nch;
    const int pt0 = (valid ? c : nch - 1) * W;
    const Loc L = locate(g, pt0);
    SChunk<T> s, s0;
    s_chunk(P, P.x, pt0, lane, L, s);
    if (dots) s_chunk(P, xs_rd, pt0, lane, L, s0);
    if (check) {   // Eq. 27 history norms before the oldest slot is overwritten
      double x2 = 0.0;
#pragma unroll
      for (int e = 0; e < W; ++e) x2 += valid ? s.I[e] * s.I[e] : 0.0;
      warp_acc(acc, nv, P.P * NSLOT + 0, x2);
      for (int jj = 0; jj < hcount; ++jj) {
        const int js = (hhead - jj + HIST_S) % HIST_S;
        double h[W];
        VT<T>::ld(P.hist[js] + pt0, h);
        double d2 = 0.0;
#pragma unroll
        for (int e = 0; e < W; ++e) d2 += valid ? (s.I[e] - h[e]) * (s.I[e] - h[e]) : 0.0;
        warp_acc(acc, nv, P.P * NSLOT + 1 + js, d2);
      }
    }
    if (valid) {
      VT<T>::st(P.hist[hslot] + pt0, s.I);
      if (adapt) VT<T>::st(xs_wr + pt0, s.I);
    }
    for (int i = 0; i < P.P; ++i) {
      const SetD<T>& S = P.set[i];
      const double rho = C.rho[i], gam = C.gamma[i];
      const bool pointwise = (S.kind == K_BOUNDS || S.kind == K_DIST);
      double a_w2 = 0, a_hv = 0, a_hh = 0, a_vh = 0, a_gv = 0, a_gg = 0, a_vv = 0, a_fn = 0, a_s2 = 0;
      for (int bl = 0; bl < S.nblk; ++bl) {
        const int prim = S.prim[bl];
        const int64_t off = (int64_t)bl * g.ld + pt0;
        T yo[W], vo[W], yn[W], vn[W], wv[W], vh[W];
        VT<T>::ldT(S.y[par] + off, yo);
        VT<T>::ldT(S.v[par] + off, vo);
        T lo[W], hi[W], mm[W], y0[W], v0[W], vh0[W];
        if (S.kind == K_BOUNDS) {
          if (S.lo_vec) VT<T>::ldT(S.lo_vec + off, lo);
          if (S.hi_vec) VT<T>::ldT(S.hi_vec + off, hi);
        }
        if (S.kind == K_DIST) VT<T>::ldT(P.m + pt0, mm);
        if (dots && pointwise) {
          VT<T>::ldT(S.y[par ^ 1] + off, y0);
          VT<T>::ldT(S.v[par ^ 1] + off, v0);
        }
        if (dots) VT<T>::ldT(S.vh0 + off, vh0);
#pragma unroll
        for (int e = 0; e < W; ++e) {
          const bool pad = !valid || pad_vec(g, prim, L, e);
          const double sv = pad ? 0.0 : s.get(prim, e);
          const double yoe = (double)yo[e], voe = (double)vo[e];
          const double xbar = gam * sv + (1.0 - gam) * yoe;         // relaxation
          const double w = (double)(T)(xbar - voe / rho);
          wv[e] = pad ? (T)0 : (T)w;
          if (pointwise) {
            double y;
            if (S.kind == K_DIST) {
              y = ((double)mm[e] + rho * w) / (1.0 + rho);         // Eq. 22
            } else {
              const double l = S.lo_vec ? (double)lo[e] : S.lo;
              const double h = S.hi_vec ? (double)hi[e] : S.hi;
              y = w < l ? l : (w > h ? h : w);
              if (check && !pad) {
                const double cl = sv < l ? l : (sv > h ? h : sv);
                a_fn += (sv - cl) * (sv - cl);
              }
            }
            const double yt = (double)(T)y;
            const double vt = (double)(T)(rho * (yt - w));          // Eq. 21 as rho (y - w), L26
            yn[e] = pad ? (T)0 : (T)yt;
            vn[e] = pad ? (T)0 : (T)vt;
            if (dots && !pad) {
              const double dg = -(yt - (double)y0[e]);
              const double dv = vt - (double)v0[e];
              a_gv += dg * dv; a_gg += dg * dg; a_vv += dv * dv;
            }
          } else if (!pad) {
            a_w2 += w * w;
          }
          if (adapt) {                                               // Alg. 2 line 1
            const double vht = (double)(T)(voe + rho * (yoe - sv));
            vh[e] = pad ? (T)0 : (T)vht;
            if (dots && !pad) {
              const double dvh = vht - (double)vh0[e];
              const double dh = sv - s0.get(prim, e);
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
            if (check && S.s) {
              T sv[W];
#pragma unroll
              for (int e = 0; e < W; ++e) sv[e] = pad_vec(g, prim, L, e) ? (T)0 : (T)s.get(prim, e);
              VT<T>::stT(S.s + off, sv);
            }
          }
          if (adapt) VT<T>::stT(S.vh0 + off, vh);
        }
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
  double* stage = P.partials + (size_t)gridDim.x * nv;
  if (finish_reduction(acc, nv, P.partials, P.counter, stage, sh)) {
    for (int v = threadIdx.x; v < nv; v += BLOCK) {
      const double val = __ldcg(stage + v);
      if (v < P.P * NSLOT) C.sums[v / NSLOT][v % NSLOT] = val;
      else C.evol[v - P.P * NSLOT] = val;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
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

}  // namespace sip
