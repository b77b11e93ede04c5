// sip_zmarch.cuh -- 2.5D z-marching CG kernels (sm_100a).
//
// A CTA of 8 warps owns a (y, x) tile of TYW rows x (TXW * 32 * W) points and
// walks its z range.  Each thread keeps its chunk of the operand at planes
// z-1, z, z+1 in registers, so every element is loaded once per sweep (plus
// one halo plane per z range and two halo rows per tile); the y neighbours of
// plane z come from a double-buffered shared-memory copy of the tile, the x
// neighbours by warp shuffle (warp-edge chunks through shared memory, tile
// edges through global memory).  Arithmetic is exactly that of k_cg1v /
// k_cg2v (sip_vec.cuh), so results are identical.
//
// 2D grids (ny = 1) use the same kernels with TYW = 1: z is the row index and
// there is no y neighbour.
#pragma once
#include "sip_vec.cuh"

namespace sip {

#ifndef ZSMEM
#define ZSMEM false  // false: y neighbours from global memory (measured faster on C4); true: shared tile
#endif

// 16-byte load from shared memory
template <class T>
__device__ __forceinline__ void ldS(const T* p, T* o);
template <>
__device__ __forceinline__ void ldS<float>(const float* p, float* o) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w;
}
template <>
__device__ __forceinline__ void ldS<double>(const double* p, double* o) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  o[0] = a.x; o[1] = a.y;
}

struct ZGeo {
  int on;            // kernels usable for this grid
  int txw, tyw;      // warps along x per row segment, rows per tile
  int tiles_x, tiles_y, nzc, zc;
  int row_pts;       // points per tile row = txw * 32 * W
};

template <class T>
struct ZCtx {
  static constexpr int W = VT<T>::W;
  int warp, lane, tx, ty, y, xw0, z0, z1;   // xw0: first x of my chunk
  int x_tile0, x_tile1;                    // x range of the tile
};

template <class T>
__device__ __forceinline__ ZCtx<T> zctx(const Geo& g, const ZGeo& z) {
  constexpr int W = VT<T>::W;
  ZCtx<T> c;
  c.warp = threadIdx.x >> 5;
  c.lane = threadIdx.x & 31;
  c.tx = c.warp % z.txw;
  c.ty = c.warp / z.txw;
  int b = blockIdx.x;
  const int zci = b % z.nzc;
  b /= z.nzc;
  const int tile_x = b % z.tiles_x;
  const int tile_y = b / z.tiles_x;
  c.y = tile_y * z.tyw + c.ty;
  c.x_tile0 = tile_x * z.row_pts;
  c.x_tile1 = c.x_tile0 + z.row_pts;
  c.xw0 = c.x_tile0 + (c.tx * 32 + c.lane) * W;
  c.z0 = zci * z.zc;
  c.z1 = min(g.nz, c.z0 + z.zc);
  return c;
}

// the operand at (z, yy, my chunk): p_new = r + beta p_old (USE_P) or r
template <class T, bool USE_P>
__device__ __forceinline__ void zfetch(const Geo& g, const T* r, const T* p, T beta, int z, int yy, int x,
                                       T* o) {
  constexpr int W = VT<T>::W;
  const int pt = (z * g.ny + yy) * g.nx + x;
  T a[W];
  VT<T>::ldT(r + pt, a);
  if (USE_P) {
    T b[W];
    VT<T>::ldT(p + pt, b);
#pragma unroll
    for (int e = 0; e < W; ++e) o[e] = a[e] + beta * b[e];
  } else {
#pragma unroll
    for (int e = 0; e < W; ++e) o[e] = a[e];
  }
}
template <class T, bool USE_P>
__device__ __forceinline__ T zfetch1(const Geo& g, const T* r, const T* p, T beta, int z, int yy, int x) {
  const int pt = (z * g.ny + yy) * g.nx + x;
  return USE_P ? r[pt] + beta * p[pt] : r[pt];
}

// q = C p at plane z of my chunk; cur/prev/next = planes z, z-1, z+1;
// ym/yp = rows y-1, y+1 of plane z; xl/xr = outer x neighbours of the chunk.
// A missing neighbour is replaced by the centre value, which makes its
// difference exactly 0: the same bits as the masked form of apply_C_vec.
template <class T>
__device__ __forceinline__ void zapply(const CoefT<T>& cf, const Geo& g, bool hz, bool hy, bool hx, int z, int y,
                                       int x0, const T* cur, const T* prev, const T* next, const T* ym,
                                       const T* yp, T xl, T xr, T* q) {
  constexpr int W = VT<T>::W;
  const bool zlo = z + g.z0 >= 1, zhi = z + g.z0 < g.nz_g - 1;
  const bool ylo = y >= 1, yhi = y < g.ny - 1;
  const bool xlo = x0 >= 1, xhi = x0 + W < g.nx;
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const T p0 = cur[e];
    T v = cf.cI * p0;
    if (hz) {
      const T a = (p0 - (zlo ? prev[e] : p0)) - ((zhi ? next[e] : p0) - p0);
      v += cf.cz * a;
    }
    if (hy) {
      const T a = (p0 - (ylo ? ym[e] : p0)) - ((yhi ? yp[e] : p0) - p0);
      v += cf.cy * a;
    }
    if (hx) {
      const T left = e > 0 ? cur[e - 1] : (xlo ? xl : p0);
      const T right = e < W - 1 ? cur[e + 1] : (xhi ? xr : p0);
      v += cf.cx * ((p0 - left) - (right - p0));
    }
    q[e] = v;
  }
}

// one z sweep: MODE 1 = k_cg1 (write p_j = r + beta p_{j-1}, <p, C p>),
// MODE 2 = k_cg2 (x += alpha p, r -= alpha C p, <r, r>).  Software pipelined:
// the loads of plane z+2 (operand), z+1 (x, r, y-halo rows) are issued
// while plane z is computed.
template <class T, int MODE, bool USE_P, bool Y3D, bool YSMEM>
__device__ __forceinline__ double zsweep(const Prob<T>& P, const ZGeo& Z, const CoefT<T>& cf, const T* r,
                                         const T* p, T beta, T alpha, T* pw, T* sbuf) {
  constexpr int W = VT<T>::W;
  constexpr bool UP = USE_P && MODE == 1;
  const Geo& g = P.g;
  const ZCtx<T> c = zctx<T>(g, Z);
  const bool hz = P.has[PRIM_Z], hy = P.has[PRIM_Y], hx = P.has[PRIM_X];
  const int tyw = Z.tyw, rp = Z.row_pts;
  const int xoff = (c.tx * 32 + c.lane) * W;        // my chunk inside the tile row
  const T* src_r = MODE == 1 ? r : p;               // MODE 2 reads p directly
  const bool lo_w = YSMEM && Y3D && c.ty == 0, hi_w = YSMEM && Y3D && c.ty == tyw - 1;
  auto zero = [](T* v) {
#pragma unroll
    for (int e = 0; e < W; ++e) v[e] = 0;
  };
  auto fetch_plane = [&](int z, T* o) {
    const int gz = z + g.z0;   // planes -1 and nz are ghost planes (the z-slab halo)
    if (gz >= 0 && gz < g.nz_g && z >= -1 && z <= g.nz) zfetch<T, UP>(g, src_r, p, beta, z, c.y, c.xw0, o);
    else zero(o);
  };
  auto fetch_halo = [&](int z, int yy, T* o) {
    if (z < g.nz && yy >= 0 && yy < g.ny) zfetch<T, UP>(g, src_r, p, beta, z, yy, c.xw0, o); else zero(o);
  };
  T prev[W], cur[W], nxt[W], nxt2[W];
  fetch_plane(c.z0 - 1, prev);
  fetch_plane(c.z0, cur);
  fetch_plane(c.z0 + 1, nxt);
  T xc[W], rc[W], xn[W], rn[W];
  if (MODE == 2) {
    const int pt = (c.z0 * g.ny + c.y) * g.nx + c.xw0;
    VT<T>::ldcs(P.x + pt, xc);
    VT<T>::ldcs(P.r + pt, rc);
  }
  T hlo[W], hhi[W], hlo_n[W], hhi_n[W];
  if (lo_w) fetch_halo(c.z0, c.y - 1, hlo);
  if (hi_w) fetch_halo(c.z0, c.y + 1, hhi);
  double acc = 0.0;
  for (int z = c.z0; z < c.z1; ++z) {
    // prefetch
    fetch_plane(z + 2, nxt2);
    const bool more = z + 1 < c.z1;
    if (MODE == 2 && more) {
      const int ptn = ((z + 1) * g.ny + c.y) * g.nx + c.xw0;
      VT<T>::ldcs(P.x + ptn, xn);
      VT<T>::ldcs(P.r + ptn, rn);
    }
    if (lo_w && more) fetch_halo(z + 1, c.y - 1, hlo_n);
    if (hi_w && more) fetch_halo(z + 1, c.y + 1, hhi_n);
    const int pt0 = (z * g.ny + c.y) * g.nx + c.xw0;
    T ym[W], yp[W];
    T xl, xr;
    if (Y3D && !YSMEM) {
      // y neighbours straight from global memory (L1 / L2 hits: the adjacent
      // rows belong to the neighbouring warps of this CTA); no barrier
      fetch_halo(z, c.y - 1, ym);
      fetch_halo(z, c.y + 1, yp);
      xl = __shfl_up_sync(0xffffffffu, cur[W - 1], 1);
      xr = __shfl_down_sync(0xffffffffu, cur[0], 1);
      if (c.lane == 0 && (c.xw0 % g.nx) > 0) xl = zfetch1<T, UP>(g, src_r, p, beta, z, c.y, c.xw0 - 1);
      if (c.lane == 31 && c.xw0 + W < g.nx) xr = zfetch1<T, UP>(g, src_r, p, beta, z, c.y, c.xw0 + W);
    } else if (Y3D) {
      // tile plane in shared memory (rows 0 and tyw+1 are the y halo)
      T* sb = sbuf + (z & 1) * (tyw + 2) * rp;
      VT<T>::stT(sb + (c.ty + 1) * rp + xoff, cur);
      if (lo_w) VT<T>::stT(sb + xoff, hlo);
      if (hi_w) VT<T>::stT(sb + (tyw + 1) * rp + xoff, hhi);
      __syncthreads();
      ldS<T>(sb + c.ty * rp + xoff, ym);
      ldS<T>(sb + (c.ty + 2) * rp + xoff, yp);
      // x neighbours: shuffle inside the warp, shared memory across warps
      xl = __shfl_up_sync(0xffffffffu, cur[W - 1], 1);
      xr = __shfl_down_sync(0xffffffffu, cur[0], 1);
      if (c.lane == 0) {
        if (xoff > 0) xl = sb[(c.ty + 1) * rp + xoff - 1];
        else if (c.x_tile0 > 0) xl = zfetch1<T, UP>(g, src_r, p, beta, z, c.y, c.x_tile0 - 1);
      }
      if (c.lane == 31) {
        if (xoff + W < rp) xr = sb[(c.ty + 1) * rp + xoff + W];
        else if (c.x_tile1 < g.nx) xr = zfetch1<T, UP>(g, src_r, p, beta, z, c.y, c.x_tile1);
      }
    } else {
      xl = __shfl_up_sync(0xffffffffu, cur[W - 1], 1);
      xr = __shfl_down_sync(0xffffffffu, cur[0], 1);
      if (c.lane == 0 && c.xw0 > 0) xl = zfetch1<T, UP>(g, src_r, p, beta, z, 0, c.xw0 - 1);
      if (c.lane == 31 && c.xw0 + W < g.nx) xr = zfetch1<T, UP>(g, src_r, p, beta, z, 0, c.xw0 + W);
    }
    T q[W];
    zapply<T>(cf, g, hz, Y3D && hy, hx, z, c.y, c.xw0, cur, prev, nxt, ym, yp, xl, xr, q);
    if (MODE == 1) {
      VT<T>::stT(pw + pt0, cur);
      T s = 0;
#pragma unroll
      for (int e = 0; e < W; ++e) s += cur[e] * q[e];
      acc += (double)s;
    } else {
      T s = 0;
#pragma unroll
      for (int e = 0; e < W; ++e) {
        xc[e] = xc[e] + alpha * cur[e];
        rc[e] = rc[e] - alpha * q[e];
        s += rc[e] * rc[e];
      }
      VT<T>::stT(P.x + pt0, xc);
      VT<T>::stT(P.r + pt0, rc);
      acc += (double)s;
    }
#pragma unroll
    for (int e = 0; e < W; ++e) {
      prev[e] = cur[e]; cur[e] = nxt[e]; nxt[e] = nxt2[e];
      if (MODE == 2) { xc[e] = xn[e]; rc[e] = rn[e]; }
      if (lo_w) hlo[e] = hlo_n[e];
      if (hi_w) hhi[e] = hhi_n[e];
    }
  }
  return acc;
}

template <class T, bool Y3D>
__global__ void __launch_bounds__(BLOCK) k_cg1z(const __grid_constant__ Prob<T> P, const __grid_constant__ ZGeo Z,
                                               int j) {
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  const Geo& g = P.g;
  if (j == 0 && C.zero_x) {   // b = 0 gives x = 0
    const int nch = g.N / W;
    for (int c = blockIdx.x * BLOCK + threadIdx.x; c < nch; c += gridDim.x * BLOCK) {
      T z[W] = {};
      VT<T>::stT(P.x + c * W, z);
    }
    return;
  }
  if (!C.cg_active) return;
  extern __shared__ __align__(16) unsigned char zsm[];
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  const CoefT<T> cf(C);
  const T beta = (T)C.beta;
  const T* pold = j > 0 ? p_slot(P, j - 1) : nullptr;
  T* pw = p_slot(P, j);
  double pq = j > 0 ? zsweep<T, 1, true, Y3D, ZSMEM>(P, Z, cf, P.r, pold, beta, (T)0, pw, (T*)zsm)
                    : zsweep<T, 1, false, Y3D, ZSMEM>(P, Z, cf, P.r, pold, beta, (T)0, pw, (T*)zsm);
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

template <class T, bool Y3D>
__global__ void __launch_bounds__(BLOCK) k_cg2z(const __grid_constant__ Prob<T> P, const __grid_constant__ ZGeo Z,
                                               int j) {
  Ctrl& C = *P.ctrl;
  if (C.stopped || !C.cg_active) return;
  extern __shared__ __align__(16) unsigned char zsm[];
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  const CoefT<T> cf(C);
  const T alpha = (T)C.alpha;
  double rr = zsweep<T, 2, false, Y3D, ZSMEM>(P, Z, cf, nullptr, P.pb[j & 1], (T)0, alpha, nullptr, (T*)zsm);
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

}  // namespace sip
