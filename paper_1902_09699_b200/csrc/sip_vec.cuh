// sip_vec.cuh -- vectorised stencil kernels for the x-update (sm_100a).
//
// Each thread owns W = 16 / sizeof(T) consecutive x points ("chunk": one
// 128-bit load per array).  Chunks of a warp are consecutive, so the x
// neighbours come from the adjacent lanes by shuffle (lanes 0 / 31 load their
// outer neighbour); the y and z neighbours are 128-bit loads of the adjacent
// rows / planes, issued unconditionally (the ghost planes of every N-field
// make the out-of-domain addresses valid) and masked afterwards.  Requires
// nx % W == 0; the scalar kernels of sip_kernels.cuh cover the general case.
//
// Precision (reading L20): per-point arithmetic is done in the storage type T
// (fp32 for the fp32 configs, as the paper's Float32 runs); every
// reduction is accumulated in fp64 and every scalar (alpha, beta, rho, the
// coefficients of C) is kept in fp64 in the control block.
#pragma once
#include "sip_kernels.cuh"

#ifndef CG2_MINB
#define CG2_MINB 3
#endif
namespace sip {

template <class T> struct VT;
template <> struct VT<float> {
  static constexpr int W = 4;
  __device__ static void ldT(const float* p, float* o) {
    float4 a = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  }
  __device__ static void ldcs(const float* p, float* o) {   // coherent, streaming
    float4 a = __ldcs(reinterpret_cast<const float4*>(p));
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  }
  __device__ static void stT(float* p, const float* o) {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
  }
  __device__ static void ldT_s(const float* p, float* o) {   // shared memory
    float4 a = *reinterpret_cast<const float4*>(p);
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
  }
  // double helpers (used by the set passes where the math stays in fp64)
  __device__ static void ld(const float* p, double* o) {
    float t[4]; ldT(p, t);
    o[0] = t[0]; o[1] = t[1]; o[2] = t[2]; o[3] = t[3];
  }
  __device__ static void st(float* p, const double* o) {
    float t[4] = {(float)o[0], (float)o[1], (float)o[2], (float)o[3]};
    stT(p, t);
  }
};
template <> struct VT<double> {
  static constexpr int W = 2;
  __device__ static void ldT(const double* p, double* o) {
    double2 a = __ldg(reinterpret_cast<const double2*>(p));
    o[0] = a.x; o[1] = a.y;
  }
  __device__ static void ldcs(const double* p, double* o) {
    double2 a = __ldcs(reinterpret_cast<const double2*>(p));
    o[0] = a.x; o[1] = a.y;
  }
  __device__ static void stT(double* p, const double* o) {
    *reinterpret_cast<double2*>(p) = make_double2(o[0], o[1]);
  }
  __device__ static void ldT_s(const double* p, double* o) {   // shared memory
    double2 a = *reinterpret_cast<const double2*>(p);
    o[0] = a.x; o[1] = a.y;
  }
  __device__ static void ld(const double* p, double* o) { ldT(p, o); }
  __device__ static void st(double* p, const double* o) { stT(p, o); }
};

template <class T>
struct CoefT {
  T cI, cz, cy, cx;
  __device__ explicit CoefT(const Ctrl& C) : cI((T)C.cI), cz((T)C.cz), cy((T)C.cy), cx((T)C.cx) {}
};

// k_cgx: the deferred x update after the CG loop, x += sum_j alpha_j p_j
// over the cg_count completed steps, in step order (Eq. 21 line 1's CG)
template <class T>
__global__ void __launch_bounds__(BLOCK) k_cgx(const __grid_constant__ Prob<T> P) {
  pdl_begin();
  constexpr int W = VT<T>::W;
  const Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  const int n = C.cg_count;
  if (n == 0) return;
  T al[MAXCG];
#pragma unroll
  for (int j = 0; j < MAXCG; ++j) al[j] = (T)C.alph[j];
  const int nch = P.g.N / W;
  for (int c = blockIdx.x * BLOCK + threadIdx.x; c < nch; c += gridDim.x * BLOCK) {
    const int pt0 = c * W;
    T xv[W];
    VT<T>::ldcs(P.x + pt0, xv);
#pragma unroll
    for (int j = 0; j < MAXCG; ++j) {
      if (j >= n) break;
      T pv[W];
      VT<T>::ldcs(P.pr[j] + pt0, pv);
#pragma unroll
      for (int e = 0; e < W; ++e) xv[e] = xv[e] + al[j] * pv[e];
    }
    VT<T>::stT(P.x + pt0, xv);
  }
}

// ------------------------------------------------------------ lean flat CG
// One thread per chunk, grid-stride, no shuffles.  C p at the chunk in the
// difference form of apply_C_vec / zapply: per axis a = (p0 - m) - (n - p0)
// with an absent neighbour replaced by p0 (its difference is exactly 0), so
// no large terms cancel (fp32 fields of ~10^3 keep their digits); the masks
// are computed once per chunk.
template <class T>
struct CGLoc {   // chunk location: which neighbours exist
  bool zlo, zhi, ylo, yhi, xlo, xhi;
  T cI, cz, cy, cx;
  __device__ __forceinline__ CGLoc(const Geo& g, const CoefT<T>& k, int c, int ncr, const FastDiv& dncr) {
    const int row = (int)dncr.div((uint32_t)c);
    const int xc = c - row * ncr;
    const int iz = g.ny > 1 ? (int)g.dny.div((uint32_t)row) : row;
    const int iy = row - iz * g.ny;
    const int gz = iz + g.z0;
    zlo = gz >= 1; zhi = gz < g.nz_g - 1;
    ylo = iy >= 1; yhi = iy < g.ny - 1;
    xlo = xc > 0; xhi = xc < ncr - 1;
    cI = k.cI; cz = k.cz; cy = k.cy; cx = k.cx;
  }
  template <int W>
  __device__ __forceinline__ void apply(const T* cur, const T* zm, const T* zp, const T* ym, const T* yp, T xl,
                                        T xr, bool hy, T* q) const {
#pragma unroll
    for (int e = 0; e < W; ++e) {
      const T p0 = cur[e];
      T v = cI * p0;
      v += cz * ((p0 - (zlo ? zm[e] : p0)) - ((zhi ? zp[e] : p0) - p0));
      if (hy) v += cy * ((p0 - (ylo ? ym[e] : p0)) - ((yhi ? yp[e] : p0) - p0));
      const T left = e > 0 ? cur[e - 1] : (xlo ? xl : p0);
      const T right = e < W - 1 ? cur[e + 1] : (xhi ? xr : p0);
      v += cx * ((p0 - left) - (right - p0));
      q[e] = v;
    }
  }
};

template <class T>
__device__ __forceinline__ CoefT<T> coefs_present(const Prob<T>& P, const Ctrl& C) {
  CoefT<T> k(C);
  if (!P.has[PRIM_Z]) k.cz = (T)0;
  if (!P.has[PRIM_Y] || P.g.ny == 1) k.cy = (T)0;
  if (!P.has[PRIM_X]) k.cx = (T)0;
  return k;
}

// plain (coherent) or read-only-path loads: the single-CTA CG re-reads in
// the same kernel what other threads wrote
template <class T, bool NC>
__device__ __forceinline__ void ldv(const T* p, T* o) {
  if (NC) VT<T>::ldT(p, o);
  else VT<T>::ldT_s(p, o);
}

// Energy form of k_cg1's dot: C = c_I I + sum_a c_a D_a^T D_a (+ c_F G^T S G,
// the ub term), so <p, C p> = c_I ||p||^2 + sum_a c_a ||D_a p||^2 (+ <p, ub>).
// Each chunk adds its points' forward differences (the pair (i, i+1) belongs
// to i, absent when i is the last point of the axis), so only the z+1, y+1
// and x+1 neighbours of p_j are rebuilt from r and p_{j-1} (3 instead of 7
// positions; every term is >= 0, nothing cancels).  p_j -> ring slot j.
template <class T, bool HY, bool NC>
__device__ __forceinline__ double cg1e_chunks(const Prob<T>& P, const Ctrl& C, int j, int c_first, int c_step) {
  constexpr int W = VT<T>::W;
  const Geo& g = P.g;
  const int nch = g.N / W;
  const CoefT<T> k = coefs_present(P, C);
  const T beta = (T)C.beta;
  const bool usep = j > 0;
  const T* r = P.r;
  const T* po = usep ? p_slot(P, j - 1) : P.r;
  T* pw = p_slot(P, j);
  const int ncr = g.nx / W;
  FastDiv dncr;
  dncr.d = P.dncr.d; dncr.m = P.dncr.m; dncr.l = P.dncr.l;
  const int pl = g.plane, nx = g.nx;
  double pq = 0.0;
#pragma unroll 1
  for (int c = c_first; c < nch; c += c_step) {
    const int pt0 = c * W;
    const CGLoc<T> L(g, k, c, ncr, dncr);
    T a0[W], az[W], ay[W], b0[W], bz[W], by[W];
    ldv<T, NC>(r + pt0, a0);
    ldv<T, NC>(r + pt0 + pl, az);
    if (HY) ldv<T, NC>(r + pt0 + nx, ay);
    T ar = r[pt0 + W];
    if (usep) {
      ldv<T, NC>(po + pt0, b0);
      ldv<T, NC>(po + pt0 + pl, bz);
      if (HY) ldv<T, NC>(po + pt0 + nx, by);
      const T br = po[pt0 + W];
#pragma unroll
      for (int e = 0; e < W; ++e) {
        a0[e] = a0[e] + beta * b0[e];
        az[e] = az[e] + beta * bz[e];
        if (HY) ay[e] = ay[e] + beta * by[e];
      }
      ar = ar + beta * br;
    }
    VT<T>::stT(pw + pt0, a0);
    T sI = 0, sz = 0, sy = 0, sx = 0;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      sI += a0[e] * a0[e];
      const T dz = az[e] - a0[e];
      sz += dz * dz;
      if (HY) { const T dy = ay[e] - a0[e]; sy += dy * dy; }
      if (e < W - 1) { const T dx = a0[e + 1] - a0[e]; sx += dx * dx; }
    }
    {
      const T dx = ar - a0[W - 1];
      if (L.xhi) sx += dx * dx;
    }
    T s = L.cI * sI + (L.zhi ? L.cz * sz : (T)0) + L.cx * sx;
    if (HY && L.yhi) s += L.cy * sy;
    if (P.ub) {   // the data operator's term, c_F G^T S G p_j (k_blurF)
      T u[W];
      ldv<T, NC>(P.ub + pt0, u);
#pragma unroll
      for (int e = 0; e < W; ++e) s += a0[e] * u[e];
    }
    pq += (double)s;
  }
  return pq;
}

// r -= alpha C p_j and <r, r> over chunks c_first, c_first + c_step, ...
template <class T, bool HY, bool NC>
__device__ __forceinline__ double cg2_chunks(const Prob<T>& P, const Ctrl& C, int j, int c_first, int c_step) {
  constexpr int W = VT<T>::W;
  const Geo& g = P.g;
  const int nch = g.N / W;
  const CoefT<T> k = coefs_present(P, C);
  const T alpha = (T)C.alpha;
  const T* p = p_slot(P, j);
  const int ncr = g.nx / W;
  FastDiv dncr;
  dncr.d = P.dncr.d; dncr.m = P.dncr.m; dncr.l = P.dncr.l;
  const int pl = g.plane, nx = g.nx;
  double rr = 0.0;
#pragma unroll 1
  for (int c = c_first; c < nch; c += c_step) {
    const int pt0 = c * W;
    const CGLoc<T> L(g, k, c, ncr, dncr);
    T a0[W], a1[W], a2[W], a3[W], a4[W], rv[W];
    ldv<T, NC>(p + pt0, a0);
    ldv<T, NC>(p + pt0 - pl, a1);
    ldv<T, NC>(p + pt0 + pl, a2);
    if (HY) { ldv<T, NC>(p + pt0 - nx, a3); ldv<T, NC>(p + pt0 + nx, a4); }
    const T xl = p[pt0 - 1], xr = p[pt0 + W];
    if (NC) VT<T>::ldcs(P.r + pt0, rv);
    else VT<T>::ldT_s(P.r + pt0, rv);
    T q[W];
    L.template apply<W>(a0, a1, a2, a3, a4, xl, xr, HY, q);
    if (P.ub) {
      T u[W];
      ldv<T, NC>(P.ub + pt0, u);
#pragma unroll
      for (int e = 0; e < W; ++e) q[e] += u[e];
    }
    T s = 0;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      rv[e] = rv[e] - alpha * q[e];
      s += rv[e] * rv[e];
    }
    VT<T>::stT(P.r + pt0, rv);
    rr += (double)s;
  }
  return rr;
}

// cg1e over z pairs (see cg2p_chunks): the chunks at planes 2q and 2q + 1;
// p_j is rebuilt at planes z, z+1, z+2 (and y+1, x+1 of both), 14 loads for
// two chunks instead of 16.  Same per-point arithmetic as cg1e_chunks.
template <class T, bool HY>
__device__ __forceinline__ double cg1ep_chunks(const Prob<T>& P, const Ctrl& C, int j, int q_first, int q_step) {
  constexpr int W = VT<T>::W;
  const Geo& g = P.g;
  const CoefT<T> k = coefs_present(P, C);
  const T beta = (T)C.beta;
  const bool usep = j > 0;
  const T* r = P.r;
  const T* po = usep ? p_slot(P, j - 1) : P.r;
  T* pw = p_slot(P, j);
  const int ncr = g.nx / W;
  FastDiv dncr;
  dncr.d = P.dncr.d; dncr.m = P.dncr.m; dncr.l = P.dncr.l;
  const int pl = g.plane, nx = g.nx;
  const int cpp = pl / W;
  const int npair = ((g.nz + 1) >> 1) * cpp;
  double pq = 0.0;
#pragma unroll 1
  for (int q = q_first; q < npair; q += q_step) {
    const int zp = (int)g.dplane.div((uint32_t)(q * W));
    const int c = q + zp * cpp;
    const bool two = 2 * zp + 1 < g.nz;
    const int pt0 = c * W, pt1 = pt0 + pl;
    const CGLoc<T> L(g, k, c, ncr, dncr);
    const bool zhi1 = 2 * zp + 1 + g.z0 < g.nz_g - 1;
    T a0[W], a1[W], a2[W], y0[W], y1[W];
    VT<T>::ldT(r + pt0, a0);
    VT<T>::ldT(r + pt1, a1);
    VT<T>::ldT(r + pt1 + pl, a2);
    if (HY) { VT<T>::ldT(r + pt0 + nx, y0); VT<T>::ldT(r + pt1 + nx, y1); }
    T x0 = r[pt0 + W], x1 = r[pt1 + W];
    if (usep) {
      T b0[W], b1[W], b2[W], c0[W], c1[W];
      VT<T>::ldT(po + pt0, b0);
      VT<T>::ldT(po + pt1, b1);
      VT<T>::ldT(po + pt1 + pl, b2);
      if (HY) { VT<T>::ldT(po + pt0 + nx, c0); VT<T>::ldT(po + pt1 + nx, c1); }
      const T bx0 = po[pt0 + W], bx1 = po[pt1 + W];
#pragma unroll
      for (int e = 0; e < W; ++e) {
        a0[e] = a0[e] + beta * b0[e];
        a1[e] = a1[e] + beta * b1[e];
        a2[e] = a2[e] + beta * b2[e];
        if (HY) { y0[e] = y0[e] + beta * c0[e]; y1[e] = y1[e] + beta * c1[e]; }
      }
      x0 = x0 + beta * bx0;
      x1 = x1 + beta * bx1;
    }
    VT<T>::stT(pw + pt0, a0);
    if (two) VT<T>::stT(pw + pt1, a1);
    // chunk 0 (plane z): z pair with a1; chunk 1 (plane z+1): z pair with a2
    T sI0 = 0, sz0 = 0, sy0 = 0, sx0 = 0, sI1 = 0, sz1 = 0, sy1 = 0, sx1 = 0;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      sI0 += a0[e] * a0[e];
      sI1 += a1[e] * a1[e];
      const T d0 = a1[e] - a0[e], d1 = a2[e] - a1[e];
      sz0 += d0 * d0;
      sz1 += d1 * d1;
      if (HY) {
        const T e0 = y0[e] - a0[e], e1 = y1[e] - a1[e];
        sy0 += e0 * e0;
        sy1 += e1 * e1;
      }
      if (e < W - 1) {
        const T f0 = a0[e + 1] - a0[e], f1 = a1[e + 1] - a1[e];
        sx0 += f0 * f0;
        sx1 += f1 * f1;
      }
    }
    if (L.xhi) {
      const T f0 = x0 - a0[W - 1], f1 = x1 - a1[W - 1];
      sx0 += f0 * f0;
      sx1 += f1 * f1;
    }
    T s0 = L.cI * sI0 + (L.zhi ? L.cz * sz0 : (T)0) + L.cx * sx0;
    T s1 = L.cI * sI1 + (zhi1 ? L.cz * sz1 : (T)0) + L.cx * sx1;
    if (HY && L.yhi) { s0 += L.cy * sy0; s1 += L.cy * sy1; }
    if (P.ub) {
      T u[W];
      VT<T>::ldT(P.ub + pt0, u);
#pragma unroll
      for (int e = 0; e < W; ++e) s0 += a0[e] * u[e];
      if (two) {
        VT<T>::ldT(P.ub + pt1, u);
#pragma unroll
        for (int e = 0; e < W; ++e) s1 += a1[e] * u[e];
      }
    }
    pq += (double)s0;
    if (two) pq += (double)s1;
  }
  return pq;
}

// cg2 over z pairs: one thread takes the chunk at plane 2q and the one above
// it (plane 2q + 1), so the four planes z-1 .. z+2 of p serve both stencils
// (14 loads for two chunks instead of 16) and two chunks' loads are in flight
// per thread.  Same per-point arithmetic as cg2_chunks.
template <class T, bool HY>
__device__ __forceinline__ double cg2p_chunks(const Prob<T>& P, const Ctrl& C, int j, int q_first, int q_step) {
  constexpr int W = VT<T>::W;
  const Geo& g = P.g;
  const CoefT<T> k = coefs_present(P, C);
  const T alpha = (T)C.alpha;
  const T* p = p_slot(P, j);
  const int ncr = g.nx / W;
  FastDiv dncr;
  dncr.d = P.dncr.d; dncr.m = P.dncr.m; dncr.l = P.dncr.l;
  const int pl = g.plane, nx = g.nx;
  const int cpp = pl / W;                    // chunks per plane
  const int npair = ((g.nz + 1) >> 1) * cpp;
  double rr = 0.0;
#pragma unroll 1
  for (int q = q_first; q < npair; q += q_step) {
    const int zp = (int)g.dplane.div((uint32_t)(q * W));   // plane pair
    const int c = q + zp * cpp;                            // chunk at plane 2 zp
    const bool two = 2 * zp + 1 < g.nz;
    const int pt0 = c * W, pt1 = pt0 + pl;
    const CGLoc<T> L(g, k, c, ncr, dncr);
    CGLoc<T> L1 = L;
    L1.zlo = true;
    L1.zhi = 2 * zp + 1 + g.z0 < g.nz_g - 1;
    T zm[W], a0[W], a1[W], z2[W], y0m[W], y0p[W], y1m[W], y1p[W], r0[W], r1[W] = {};
    VT<T>::ldT(p + pt0 - pl, zm);
    VT<T>::ldT(p + pt0, a0);
    VT<T>::ldT(p + pt1, a1);
    VT<T>::ldT(p + pt1 + pl, z2);
    if (HY) {
      VT<T>::ldT(p + pt0 - nx, y0m); VT<T>::ldT(p + pt0 + nx, y0p);
      VT<T>::ldT(p + pt1 - nx, y1m); VT<T>::ldT(p + pt1 + nx, y1p);
    }
    const T xl0 = p[pt0 - 1], xr0 = p[pt0 + W], xl1 = p[pt1 - 1], xr1 = p[pt1 + W];
    VT<T>::ldcs(P.r + pt0, r0);
    if (two) VT<T>::ldcs(P.r + pt1, r1);
    T q0[W], q1[W];
    L.template apply<W>(a0, zm, a1, y0m, y0p, xl0, xr0, HY, q0);
    L1.template apply<W>(a1, a0, z2, y1m, y1p, xl1, xr1, HY, q1);
    if (P.ub) {
      T u[W];
      VT<T>::ldT(P.ub + pt0, u);
#pragma unroll
      for (int e = 0; e < W; ++e) q0[e] += u[e];
      if (two) {
        VT<T>::ldT(P.ub + pt1, u);
#pragma unroll
        for (int e = 0; e < W; ++e) q1[e] += u[e];
      }
    }
    T s0 = 0, s1 = 0;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      r0[e] = r0[e] - alpha * q0[e];
      s0 += r0[e] * r0[e];
      r1[e] = r1[e] - alpha * q1[e];
      s1 += r1[e] * r1[e];
    }
    VT<T>::stT(P.r + pt0, r0);
    rr += (double)s0;
    if (two) {
      VT<T>::stT(P.r + pt1, r1);
      rr += (double)s1;
    }
  }
  return rr;
}

// k_cg1f(j): p_j = r + beta p_{j-1} (p_0 = r) and <p_j, C p_j>; p_j -> slot j
template <class T, bool HY>
__global__ void __launch_bounds__(BLOCK, 4) k_cg1f(const __grid_constant__ Prob<T> P, int j) {
  pdl_begin();
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  const Geo& g = P.g;
  const int nch = g.N / W;
  if (j == 0 && C.zero_x) {   // b = 0 gives x = 0
    for (int c = blockIdx.x * BLOCK + threadIdx.x; c < nch; c += gridDim.x * BLOCK) {
      T z[W] = {};
      VT<T>::stT(P.x + c * W, z);
    }
    return;
  }
  if (!C.cg_active) return;
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  double pq = cg1ep_chunks<T, HY>(P, C, j, blockIdx.x * BLOCK + threadIdx.x, gridDim.x * BLOCK);
  pq = block_sum(pq, sh);
  if (threadIdx.x == 0) P.partials[blockIdx.x] = pq;
  if (last_block(P.counter)) {
    reduce_partials(P.partials, 1, out, sh);
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      if (P.nranks > 1) publish(P, out, 1, 0, 1);
      else fin_cg1(C, out, j);
    }
  }
}

// k_cg2f(j): r -= alpha C p_j and <r, r> (the x update is deferred to k_cgx)
template <class T, bool HY>
__global__ void __launch_bounds__(BLOCK, CG2_MINB) k_cg2f(const __grid_constant__ Prob<T> P, int j) {
  pdl_begin();
  Ctrl& C = *P.ctrl;
  if (C.stopped || !C.cg_active) return;
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  double rr = cg2p_chunks<T, HY>(P, C, j, blockIdx.x * BLOCK + threadIdx.x, gridDim.x * BLOCK);
  rr = block_sum(rr, sh);
  if (threadIdx.x == 0) P.partials[blockIdx.x] = rr;
  if (last_block(P.counter)) {
    reduce_partials(P.partials, 1, out, sh);
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      if (P.nranks > 1) publish(P, out, 1, 0, 1);
      else fin_cg2(C, out, j);
    }
  }
}

// k_cgsmall: the whole CG loop of a small grid (one rank) in ONE CTA, the
// block barrier in place of the kernel boundaries: the same chunk bodies,
// block sums and finalisers (fin_cg1 / fin_cg2, Eq. 25) as k_cg1f / k_cg2f,
// 2 n_cg launches -> 1 (C1 and the tiny cases are latency-bound)
template <class T, bool HY>
__global__ void __launch_bounds__(BLOCK) k_cgsmall(const __grid_constant__ Prob<T> P, int n_cg) {
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  __shared__ double sh[NWARP + 1];
  const int nch = P.g.N / W;
  if (C.zero_x) {   // b = 0 gives x = 0
    for (int c = threadIdx.x; c < nch; c += BLOCK) {
      T z[W] = {};
      VT<T>::stT(P.x + c * W, z);
    }
    return;
  }
  for (int j = 0; j < n_cg; ++j) {
    if (!C.cg_active) break;
    double pq = cg1e_chunks<T, HY, false>(P, C, j, threadIdx.x, BLOCK);
    pq = block_sum(pq, sh);
    if (threadIdx.x == 0) fin_cg1(C, &pq, j);
    __syncthreads();
    if (!C.cg_active) break;
    double rr = cg2_chunks<T, HY, false>(P, C, j, threadIdx.x, BLOCK);
    rr = block_sum(rr, sh);
    if (threadIdx.x == 0) fin_cg2(C, &rr, j);
    __syncthreads();
  }
}

// k_rhsp: the vectorised rhs (Eq. 21 line 1, Eq. 25): b = sum_i A_i^T
// (rho_i y_i + v_i), r = b - C x, ||b||^2, ||r||^2.  Every field stores 0 at
// the entries an operator block does not have (pads) and in the ghost
// planes, so the transposed differences need no masks: D^T u at a point is
// u(point - 1 step) - u(point), whose absent terms read those zeros (reading
// L3).  Over z pairs (the chunks at planes 2q and 2q + 1, as the CG
// kernels): a D_z block's u at plane z serves as the lower neighbour of the
// chunk above, x's planes z-1 .. z+2 serve both stencils, and every block's
// loads for two chunks are in flight together (measured: C4 rhs 1.09 ->
// 0.93 ms per step, C5-L1 9.9 -> 7.9 ms, against one chunk per thread).
#ifndef RHS_MINB
#define RHS_MINB 3
#endif
template <class T, bool HY>
__global__ void __launch_bounds__(BLOCK, RHS_MINB) k_rhsp(const __grid_constant__ Prob<T> P) {
  pdl_begin();
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  __shared__ double sh[NWARP + 1];
  __shared__ double out[2];
  const Geo& g = P.g;
  const int par = C.k & 1;
  const CoefT<T> k = coefs_present(P, C);
  const int ncr = g.nx / W;
  FastDiv dncr;
  dncr.d = P.dncr.d; dncr.m = P.dncr.m; dncr.l = P.dncr.l;
  const int pl = g.plane, nx = g.nx;
  const int cpp = pl / W;
  const int npair = ((g.nz + 1) >> 1) * cpp;
  double bb = 0.0, rr = 0.0;
  for (int q = blockIdx.x * BLOCK + threadIdx.x; q < npair; q += gridDim.x * BLOCK) {
    const int zp = (int)g.dplane.div((uint32_t)(q * W));
    const int c = q + zp * cpp;
    const bool two = 2 * zp + 1 < g.nz;
    const int pt0 = c * W, pt1 = pt0 + pl;
    T b0[W], b1[W];
#pragma unroll
    for (int e = 0; e < W; ++e) { b0[e] = 0; b1[e] = 0; }
    for (int i = 0; i < P.P; ++i) {
      const SetD<T>& S = P.set[i];
      const T rho = (T)C.rho[i];
      for (int bl = 0; bl < S.nblk; ++bl) {
        const int prim = S.prim[bl];
        const T* y = S.y[par] + (int64_t)bl * g.ld + pt0;
        const T* v = S.v[par] + (int64_t)bl * g.ld + pt0;
        T y0[W], v0[W], y1[W], v1[W], u0[W], u1[W];
        if (prim == PRIM_Z || prim == PRIM_Y) {   // read again as the z / y neighbour: keep in L2
          VT<T>::ldT(y, y0); VT<T>::ldT(v, v0);
          VT<T>::ldT(y + pl, y1); VT<T>::ldT(v + pl, v1);
        } else {
          VT<T>::ldcs(y, y0); VT<T>::ldcs(v, v0);
          VT<T>::ldcs(y + pl, y1); VT<T>::ldcs(v + pl, v1);
        }
        if (prim == PRIM_Z) {                 // D_z^T u = u[z-1] - u[z]; chunk 1's u[z-1] is chunk 0's u
          T ym[W], vm[W];
          VT<T>::ldT(y - pl, ym);
          VT<T>::ldT(v - pl, vm);
          const T ih = (T)g.ihz;
#pragma unroll
          for (int e = 0; e < W; ++e) {
            u0[e] = rho * y0[e] + v0[e];
            u1[e] = rho * y1[e] + v1[e];
            b0[e] += ((rho * ym[e] + vm[e]) - u0[e]) * ih;
            b1[e] += (u0[e] - u1[e]) * ih;
          }
          continue;
        }
#pragma unroll
        for (int e = 0; e < W; ++e) { u0[e] = rho * y0[e] + v0[e]; u1[e] = rho * y1[e] + v1[e]; }
        if (prim == PRIM_I) {
#pragma unroll
          for (int e = 0; e < W; ++e) { b0[e] += u0[e]; b1[e] += u1[e]; }
        } else if (prim == PRIM_X) {        // D_x^T u = u[x-1] - u[x]
          const T ul0 = rho * y[-1] + v[-1];
          const T ul1 = rho * y[pl - 1] + v[pl - 1];
          const T ih = (T)g.ihx;
#pragma unroll
          for (int e = 0; e < W; ++e) {
            b0[e] += ((e > 0 ? u0[e - 1] : ul0) - u0[e]) * ih;
            b1[e] += ((e > 0 ? u1[e - 1] : ul1) - u1[e]) * ih;
          }
        } else {                            // D_y^T: u[y-1] - u[y]
          T ym0[W], vm0[W], ym1[W], vm1[W];
          VT<T>::ldT(y - nx, ym0); VT<T>::ldT(v - nx, vm0);
          VT<T>::ldT(y + pl - nx, ym1); VT<T>::ldT(v + pl - nx, vm1);
          const T ih = (T)g.ihy;
#pragma unroll
          for (int e = 0; e < W; ++e) {
            b0[e] += ((rho * ym0[e] + vm0[e]) - u0[e]) * ih;
            b1[e] += ((rho * ym1[e] + vm1[e]) - u1[e]) * ih;
          }
        }
      }
    }
    // r = b - C x (Eq. 25's residual at the warm start x^k)
    const CGLoc<T> L(g, k, c, ncr, dncr);
    CGLoc<T> L1 = L;
    L1.zlo = true;
    L1.zhi = 2 * zp + 1 + g.z0 < g.nz_g - 1;
    T zm[W], a0[W], a1[W], z2[W], y0m[W], y0p[W], y1m[W], y1p[W];
    VT<T>::ldT(P.x + pt0 - pl, zm);
    VT<T>::ldT(P.x + pt0, a0);
    VT<T>::ldT(P.x + pt1, a1);
    VT<T>::ldT(P.x + pt1 + pl, z2);
    if (HY) {
      VT<T>::ldT(P.x + pt0 - nx, y0m); VT<T>::ldT(P.x + pt0 + nx, y0p);
      VT<T>::ldT(P.x + pt1 - nx, y1m); VT<T>::ldT(P.x + pt1 + nx, y1p);
    }
    const T xl0 = P.x[pt0 - 1], xr0 = P.x[pt0 + W], xl1 = P.x[pt1 - 1], xr1 = P.x[pt1 + W];
    T q0[W], q1[W];
    L.template apply<W>(a0, zm, a1, y0m, y0p, xl0, xr0, HY, q0);
    L1.template apply<W>(a1, a0, z2, y1m, y1p, xl1, xr1, HY, q1);
    T sb0 = 0, sr0 = 0, sb1 = 0, sr1 = 0, r0[W], r1[W];
#pragma unroll
    for (int e = 0; e < W; ++e) {
      r0[e] = b0[e] - q0[e];
      sb0 += b0[e] * b0[e];
      sr0 += r0[e] * r0[e];
      r1[e] = b1[e] - q1[e];
      sb1 += b1[e] * b1[e];
      sr1 += r1[e] * r1[e];
    }
    VT<T>::stT(P.r + pt0, r0);
    bb += (double)sb0;
    rr += (double)sr0;
    if (two) {
      VT<T>::stT(P.r + pt1, r1);
      bb += (double)sb1;
      rr += (double)sr1;
    }
  }
  bb = block_sum(bb, sh);
  rr = block_sum(rr, sh);
  if (threadIdx.x == 0) { P.partials[blockIdx.x * 2] = bb; P.partials[blockIdx.x * 2 + 1] = rr; }
  if (last_block(P.counter)) {
    reduce_partials(P.partials, 2, out, sh);
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      if (P.nranks > 1) publish(P, out, 2, 0, 1);
      else fin_rhs(C, out);
    }
  }
}

}  // namespace sip
