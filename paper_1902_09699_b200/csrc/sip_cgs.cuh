// sip_cgs.cuh -- staged z-marching CG kernels (sm_100a).
//
// A CTA owns a tile of TY rows x TX chunks (W = 16 / sizeof(T) points per
// chunk) of the x-y plane and marches over a range of z planes.  Each plane
// of every input array is brought into shared memory by 1D bulk async copies
// (cp.async.bulk, one per tile row, or one per plane when the tile spans
// whole rows) with a one-row / one-chunk halo, double or quadruple buffered
// on mbarriers; the 7-point operator C (Eq. 23) then reads its z, y and x
// neighbours from shared memory.  Every value is loaded from global memory
// once per CTA (plus the halo), and the kernel issues a few tens of
// instructions per chunk instead of the address arithmetic, shuffles and
// predicated loads of the register-level kernels (sip_vec.cuh).
//
//   k_cg1s(j): p_j = r + beta p_{j-1} (p_0 = r) on the staged planes into a
//              3-plane ring, <p_j, C p_j>, p_j -> ring slot j (sip_kernels)
//   k_cg2s(j): r -= alpha C p_j, <r, r>  (x is updated once by k_cgx)
//
// The arithmetic per point is that of apply_C_vec / zapply (a missing
// neighbour contributes a zero difference), in the storage precision.
#pragma once
#include "sip_stage.cuh"
#include "sip_vec.cuh"

namespace sip {

struct SGeo {
  int on;
  int tx, ty;        // tile: ty rows x tx chunks (tx * ty = BLOCK)
  int tiles_x, tiles_y, nzc, zc;
  int full;          // tile rows span whole x rows: one copy per plane
  int hrow;          // y halo rows (1 in 3D, 0 in 2D)
  int rows;          // staged rows per plane: ty + 2 hrow
};

// elements of a staged plane tile (one-row / one-chunk halo)
template <class T>
__host__ __device__ inline int splane_elems(const SGeo& Z, int nx) {
  constexpr int W = VT<T>::W;
  return Z.full ? Z.rows * nx + 2 * W : Z.rows * (Z.tx + 2) * W;
}

// issue the copies of plane z (local index, may be -1 .. nz) of `src` into
// `dst` (elements laid out [ty + 2][tx + 2][W]), counted on `bar` by the
// caller's expect_tx.  Returns the bytes issued.  Thread 0 only.
template <class T>
__device__ __forceinline__ unsigned stage_plane(const Geo& g, const SGeo& Z, const T* src, int z, int y0, int x0c,
                                                T* dst, uint64_t* bar) {
  constexpr int W = VT<T>::W;
  const int rowc = Z.tx + 2;
  const unsigned rb = (unsigned)rowc * W * sizeof(T);
  const T* base = src + ((int64_t)z * g.ny + (y0 - Z.hrow)) * g.nx + (int64_t)(x0c - 1) * W;
  if (Z.full) {   // rows are contiguous: [row y0-hrow, chunk -1 .. row y0+ty-1+hrow, chunk tx]
    const unsigned b = (unsigned)((Z.rows * g.nx + 2 * W) * sizeof(T));
    bulk_g2s(dst, base, b, bar);
    return b;
  }
  for (int r = 0; r < Z.rows; ++r) bulk_g2s(dst + r * rowc * W, base + (int64_t)r * g.nx, rb, bar);
  return rb * Z.rows;
}

// element (row r, chunk c, lane e) of a staged plane; with Z.full the rows are
// packed at nx stride (one copy), else at (tx + 2) * W
template <class T>
struct SIdx {
  int rs;   // row stride (elements)
  __device__ SIdx(const Geo& g, const SGeo& Z) : rs(Z.full ? g.nx : (Z.tx + 2) * VT<T>::W) {}
  __device__ __forceinline__ int at(int r, int c) const { return r * rs + c * VT<T>::W; }
};

template <class T>
__device__ __forceinline__ void lds(const T* p, T* o) { VT<T>::ldT_s(p, o); }

// C = cI I + cz Dz'Dz + cy Dy'Dy + cx Dx'Dx (Eq. 23) written per point as
// q = diag p0 - sum_n c_n p_n over the present neighbours n: the boundary
// rows of D'D (reading L3) drop a neighbour together with its diagonal
// share.  Coefficients of absent neighbours are 0 (so a missing primitive
// costs nothing), y and x masks are per thread, the z mask per plane.
template <class T>
struct SCo {
  T cI, cz, cyl, cyh, cxl0, cxh, cx, cxhW, d0, d1, dW;   // d*: diagonal without the z part
  __device__ SCo(const Ctrl& C, const Prob<T>& P, bool ylo, bool yhi, int ix0) {
    constexpr int W = VT<T>::W;
    const Geo& g = P.g;
    cI = (T)C.cI;
    cz = P.has[PRIM_Z] ? (T)C.cz : (T)0;
    const T cy = P.has[PRIM_Y] ? (T)C.cy : (T)0;
    cx = P.has[PRIM_X] ? (T)C.cx : (T)0;
    cyl = ylo ? cy : (T)0;
    cyh = yhi ? cy : (T)0;
    cxl0 = ix0 >= 1 ? cx : (T)0;               // left neighbour of lane 0
    cxhW = ix0 + W < g.nx ? cx : (T)0;         // right neighbour of lane W-1
    cxh = cx;
    const T dy = cI + cyl + cyh;
    d0 = dy + cxl0 + cx;                        // lane 0
    d1 = dy + cx + cx;                          // inner lanes
    dW = dy + cx + cxhW;                        // lane W-1
  }
};

template <class T, bool HY>
__device__ __forceinline__ void stencil_s(const SCo<T>& k, T czl, T czh, const T* pm, const T* pc, const T* pp,
                                          int o, int rs, T* p0out, T* q) {
  constexpr int W = VT<T>::W;
  T cur[W], zm[W], zp[W], ym[W], yp[W];
  lds<T>(pc + o, cur);
  lds<T>(pm + o, zm);
  lds<T>(pp + o, zp);
  if (HY) {
    lds<T>(pc + o - rs, ym);
    lds<T>(pc + o + rs, yp);
  }
  const T xl = pc[o - 1], xr = pc[o + W];
  const T dz = czl + czh;
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const T p0 = cur[e];
    const T de = (e == 0 ? k.d0 : (e == W - 1 ? k.dW : k.d1)) + dz;
    T v = de * p0 - czl * zm[e] - czh * zp[e];
    if (HY) v = v - k.cyl * ym[e] - k.cyh * yp[e];
    const T left = e > 0 ? cur[e - 1] : xl;
    const T right = e < W - 1 ? cur[e + 1] : xr;
    v = v - (e == 0 ? k.cxl0 : k.cx) * left - (e == W - 1 ? k.cxhW : k.cx) * right;
    q[e] = v;
    p0out[e] = p0;
  }
}

// ring sizes (planes) and prefetch distances
// (one or two CTAs per SM each keep ~60 KB of plane tiles in flight)
constexpr int CG1_RS = 8;    // staged (r, p_{j-1}) planes: RS - 1 planes in flight beyond the one consumed
constexpr int CG2_RP = 12;   // staged p_j planes: z-1 .. z+1 in use, up to z + PD in flight
constexpr int CG2_PD = 8;
constexpr int CG2_RR = 8;    // staged r tiles (no halo): z .. z + RR - 1

// tile and z range of this CTA
struct STile {
  int x0c, y0, zb, ze, tx, ty;
  __device__ STile(const Geo& g, const SGeo& Z) {
    int b = blockIdx.x;
    const int zci = b % Z.nzc;
    b /= Z.nzc;
    x0c = (b % Z.tiles_x) * Z.tx;
    y0 = (b / Z.tiles_x) * Z.ty;
    zb = zci * Z.zc;
    ze = min(g.nz, zb + Z.zc);
    tx = threadIdx.x % Z.tx;
    ty = threadIdx.x / Z.tx;
  }
};

// ------------------------------------------------------------ k_cg1s
template <class T>
__global__ void __launch_bounds__(BLOCK) k_cg1s(const __grid_constant__ Prob<T> P, const __grid_constant__ SGeo Z,
                                               int j) {
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped) return;
  const Geo& g = P.g;
  if (j == 0 && C.zero_x) {   // b = 0 gives x = 0
    const int nch = g.N / W;
    for (int c = blockIdx.x * BLOCK + threadIdx.x; c < nch; c += gridDim.x * BLOCK) {
      T zz[W] = {};
      VT<T>::stT(P.x + c * W, zz);
    }
    return;
  }
  if (!C.cg_active) return;
  extern __shared__ __align__(128) unsigned char sm_[];
  __shared__ uint64_t bar[CG1_RS];
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  const int PL = splane_elems<T>(Z, g.nx);
  const int PLa = (PL + 31) / 32 * 32;            // 128-byte aligned slots (fp32)
  T* sr = reinterpret_cast<T*>(sm_);              // [CG1_RS][PLa] staged r
  T* sq = sr + CG1_RS * PLa;                       // [CG1_RS][PLa] staged p_{j-1}
  T* pn = sq + CG1_RS * PLa;                       // [3][PLa] p_j ring
  const bool usep = j > 0;
  const T beta = (T)C.beta;
  const T* pold = usep ? p_slot(P, j - 1) : nullptr;
  T* pw = p_slot(P, j);
  const bool hy = P.has[PRIM_Y] && g.ny > 1;
  const STile t(g, Z);
  const SIdx<T> I(g, Z);
  if (threadIdx.x == 0) {
    for (int s = 0; s < CG1_RS; ++s) mbar_init(&bar[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  unsigned ph = 0;
  const unsigned bytes = (unsigned)(PL * sizeof(T));
  auto issue = [&](int z) {   // planes z of r (and p_{j-1}) into staging slot z mod CG1_RS
    if (threadIdx.x == 0 && z <= t.ze) {
      const int s = (z + CG1_RS) % CG1_RS;
      mbar_expect_tx(&bar[s], usep ? 2 * bytes : bytes);
      stage_plane<T>(g, Z, P.r, z, t.y0, t.x0c, sr + s * PLa, &bar[s]);
      if (usep) stage_plane<T>(g, Z, pold, z, t.y0, t.x0c, sq + s * PLa, &bar[s]);
    }
  };
  // p_j = r + beta p_{j-1} on every staged position of plane z -> ring slot
  const int nchk = Z.rows * (Z.tx + 2);
  constexpr int MPN = 3;             // staged chunks per thread (<= (ty + 2)(tx + 2) / BLOCK + 1)
  int mo[MPN];
#pragma unroll
  for (int u = 0; u < MPN; ++u) {
    const int kk = threadIdx.x + u * BLOCK;
    const int r = kk / (Z.tx + 2), c = kk - r * (Z.tx + 2);
    mo[u] = kk < nchk ? I.at(r, c) : -1;
  }
  auto make_pn = [&](int z) {
    const int s = (z + CG1_RS) % CG1_RS;
    mbar_wait(&bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
    T* dst = pn + ((z + 3) % 3) * PLa;
    const T* a = sr + s * PLa;
    const T* q = sq + s * PLa;
#pragma unroll
    for (int u = 0; u < MPN; ++u) {
      const int o = mo[u];
      if (o < 0) continue;
      T av[W];
      lds<T>(a + o, av);
      if (usep) {
        T qv[W];
        lds<T>(q + o, qv);
#pragma unroll
        for (int e = 0; e < W; ++e) av[e] = av[e] + beta * qv[e];
      }
      VT<T>::stT(dst + o, av);   // generic store to shared
    }
  };
  for (int z = t.zb - 1; z < t.zb - 1 + CG1_RS; ++z) issue(z);   // zb-1 .. zb+RS-2
  make_pn(t.zb - 1);
  make_pn(t.zb);
  __syncthreads();
  issue(t.zb + CG1_RS - 1);          // into the slot of zb - 1
  const int iy = t.y0 + t.ty;
  const int ix0 = (t.x0c + t.tx) * W;
  const SCo<T> k(C, P, iy >= 1, iy < g.ny - 1, ix0);
  const int om = I.at(t.ty + Z.hrow, t.tx + 1);
  double pq = 0.0;
  for (int z = t.zb; z < t.ze; ++z) {
    make_pn(z + 1);
    __syncthreads();                 // ring holds z-1, z, z+1; the staging slot of plane z is free
    issue(z + CG1_RS);               // into the slot of plane z: planes z+2 .. z+RS in flight
    const int gz = z + g.z0;
    const T czl = gz >= 1 ? k.cz : (T)0, czh = gz < g.nz_g - 1 ? k.cz : (T)0;
    T p0[W], qv[W];
    const T* r0 = pn + ((z + 2) % 3) * PLa;
    const T* r1 = pn + (z % 3) * PLa;
    const T* r2 = pn + ((z + 1) % 3) * PLa;
    if (hy) stencil_s<T, true>(k, czl, czh, r0, r1, r2, om, I.rs, p0, qv);
    else stencil_s<T, false>(k, czl, czh, r0, r1, r2, om, I.rs, p0, qv);
    VT<T>::stT(pw + ((int64_t)z * g.ny + iy) * g.nx + ix0, p0);
    T s = 0;
#pragma unroll
    for (int e = 0; e < W; ++e) s += p0[e] * qv[e];
    pq += (double)s;
    __syncthreads();                 // ring slot of z - 1 is overwritten next step
  }
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

// ------------------------------------------------------------ k_cg2s
template <class T>
__global__ void __launch_bounds__(BLOCK) k_cg2s(const __grid_constant__ Prob<T> P, const __grid_constant__ SGeo Z,
                                               int j) {
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped || !C.cg_active) return;
  extern __shared__ __align__(128) unsigned char sm_[];
  __shared__ uint64_t bar[CG2_RP];
  __shared__ uint64_t barr[CG2_RR];
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  const Geo& g = P.g;
  const int PL = splane_elems<T>(Z, g.nx);
  const int PLa = (PL + 31) / 32 * 32;
  const int RL = Z.ty * Z.tx * W;                  // r tile (no halo)
  T* sp = reinterpret_cast<T*>(sm_);               // [CG2_RP][PLa] staged p_j
  T* srr = sp + CG2_RP * PLa;                      // [CG2_RR][RL] staged r
  const T* pv = p_slot(P, j);
  const T alpha = (T)C.alpha;
  const bool hy = P.has[PRIM_Y] && g.ny > 1;
  const STile t(g, Z);
  const SIdx<T> I(g, Z);
  if (threadIdx.x == 0) {
    for (int s = 0; s < CG2_RP; ++s) mbar_init(&bar[s], 1);
    for (int s = 0; s < CG2_RR; ++s) mbar_init(&barr[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  unsigned ph = 0, phr = 0;
  const unsigned pbytes = (unsigned)(PL * sizeof(T));
  auto issue_p = [&](int z) {
    if (threadIdx.x == 0 && z <= t.ze) {
      const int s = (z + CG2_RP) % CG2_RP;
      mbar_expect_tx(&bar[s], pbytes);
      stage_plane<T>(g, Z, pv, z, t.y0, t.x0c, sp + s * PLa, &bar[s]);
    }
  };
  auto wait_p = [&](int z) {
    const int s = (z + CG2_RP) % CG2_RP;
    mbar_wait(&bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
  };
  auto issue_r = [&](int z) {   // the r tile of plane z (no halo): ty row copies, or one
    if (threadIdx.x == 0 && z < t.ze) {
      const int s = z % CG2_RR;
      const unsigned rb = (unsigned)(Z.tx * W * sizeof(T));
      mbar_expect_tx(&barr[s], rb * Z.ty);
      const T* base = P.r + ((int64_t)z * g.ny + t.y0) * g.nx + (int64_t)t.x0c * W;
      if (Z.full) bulk_g2s(srr + s * RL, base, rb * Z.ty, &barr[s]);
      else
        for (int r = 0; r < Z.ty; ++r) bulk_g2s(srr + s * RL + r * Z.tx * W, base + (int64_t)r * g.nx, rb, &barr[s]);
    }
  };
  auto wait_r = [&](int z) {
    const int s = z % CG2_RR;
    mbar_wait(&barr[s], (phr >> s) & 1u);
    phr ^= 1u << s;
  };
  for (int z = t.zb - 1; z <= t.zb + CG2_PD - 1; ++z) issue_p(z);   // z-1 .. z+PD-1
  for (int z = t.zb; z < t.zb + CG2_RR - 1; ++z) issue_r(z);
  wait_p(t.zb - 1);
  wait_p(t.zb);
  const int iy = t.y0 + t.ty;
  const int ix0 = (t.x0c + t.tx) * W;
  const SCo<T> k(C, P, iy >= 1, iy < g.ny - 1, ix0);
  const int om = I.at(t.ty + Z.hrow, t.tx + 1);
  const int orr = (t.ty * Z.tx + t.tx) * W;
  double rr = 0.0;
  for (int z = t.zb; z < t.ze; ++z) {
    issue_p(z + CG2_PD);             // slot of z + PD - RP <= z - 2: free since the last step's barrier
    issue_r(z + CG2_RR - 1);         // slot of z - 1: free
    wait_p(z + 1);
    wait_r(z);
    const int gz = z + g.z0;
    const T czl = gz >= 1 ? k.cz : (T)0, czh = gz < g.nz_g - 1 ? k.cz : (T)0;
    T p0[W], qv[W], rv[W];
    const T* r0 = sp + ((z - 1 + CG2_RP) % CG2_RP) * PLa;
    const T* r1 = sp + (z % CG2_RP) * PLa;
    const T* r2 = sp + ((z + 1) % CG2_RP) * PLa;
    if (hy) stencil_s<T, true>(k, czl, czh, r0, r1, r2, om, I.rs, p0, qv);
    else stencil_s<T, false>(k, czl, czh, r0, r1, r2, om, I.rs, p0, qv);
    lds<T>(srr + (z % CG2_RR) * RL + orr, rv);
    T s = 0;
#pragma unroll
    for (int e = 0; e < W; ++e) {
      rv[e] = rv[e] - alpha * qv[e];
      s += rv[e] * rv[e];
    }
    VT<T>::stT(P.r + ((int64_t)z * g.ny + iy) * g.nx + ix0, rv);
    rr += (double)s;
    __syncthreads();
  }
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

// dynamic shared memory (bytes) of the staged CG kernels
template <class T>
__host__ inline size_t cgs_smem(const SGeo& Z, int nx, bool cg1) {
  constexpr int W = VT<T>::W;
  const int PL = splane_elems<T>(Z, nx);
  const int PLa = (PL + 31) / 32 * 32;
  const int RL = Z.ty * Z.tx * W;
  return cg1 ? (size_t)(2 * CG1_RS + 3) * PLa * sizeof(T) : ((size_t)CG2_RP * PLa + (size_t)CG2_RR * RL) * sizeof(T);
}

}  // namespace sip
