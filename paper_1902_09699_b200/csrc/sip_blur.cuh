// sip_blur.cuh -- the data operator's term of C p on the vectorised CG path
// (C3: F = S G, a 5x5 Gaussian G restricted to the observed pixels S; P:39,
// P:613, reading L21).  When the kernel is separable (K = g_z g_x^T, checked
// at setup), one tiled kernel per CG step forms
//     u = c_F G^T (S (G p_j)),   p_j = r + beta p_{j-1}
// on a TZ x TX tile in shared memory: p_j on the tile with a 2 r halo (zero
// outside the grid: 'same' zero padding), a row pass and a column pass for
// G (kz + kx FMAs per point instead of kz kx), the mask, then the same two
// passes with the mirrored taps for G^T.  k_cg1f / k_cg2f add u[pt] to the
// stencil part of C p.
#pragma once
#include "sip_kernels.cuh"

namespace sip {

constexpr int BF_TZ = 16, BF_TX = 64;   // interior tile (points); 256 threads

__host__ __device__ inline int bf_halo_z(int kh) { return 2 * (kh / 2); }
__host__ __device__ inline int bf_halo_x(int kw) { return 2 * (kw / 2); }
__host__ inline size_t blurf_smem(int kh, int kw, size_t word) {
  const int hz = bf_halo_z(kh), hx = bf_halo_x(kw);
  const int pz = BF_TZ + 2 * hz, px = BF_TX + 2 * hx;           // p_j
  const int sz = BF_TZ + hz, sx = BF_TX + hx;                   // S G p (interior + one radius)
  return word * ((size_t)pz * px + (size_t)pz * sx + (size_t)sz * sx + (size_t)sz * BF_TX);
}

template <class T>
__global__ void __launch_bounds__(BLOCK) k_blurF(const __grid_constant__ Prob<T> P, int j) {
  const Ctrl& C = *P.ctrl;
  if (C.stopped || !C.cg_active) return;
  extern __shared__ __align__(16) unsigned char bf_raw[];
  T* bf = reinterpret_cast<T*>(bf_raw);   // the grid's precision (fp64 runs stay fp64)
  const Geo& g = P.g;
  const int rz = g.kh / 2, rx = g.kw / 2;
  const int hz = 2 * rz, hx = 2 * rx;
  const int pz = BF_TZ + 2 * hz, px = BF_TX + 2 * hx;
  const int sz = BF_TZ + 2 * rz, sx = BF_TX + 2 * rx;
  T* sp = bf;                           // [pz][px]   p_j
  T* h1 = sp + pz * px;                 // [pz][sx]   row pass of G
  T* ss = h1 + pz * sx;                 // [sz][sx]   S G p
  T* h2 = ss + sz * sx;                 // [sz][TX]   row pass of G^T
  const T beta = (T)C.beta;
  const bool usep = j > 0;
  const T* r = P.r;
  const T* po = usep ? p_slot(P, j - 1) : P.r;
  const int tiles_x = (g.nx + BF_TX - 1) / BF_TX;
  const int tiles = tiles_x * ((g.nz + BF_TZ - 1) / BF_TZ);
  const T cF = (T)C.cF;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int z0 = (t / tiles_x) * BF_TZ, x0 = (t % tiles_x) * BF_TX;
    // p_j on the tile + 2 r halo, zero outside the grid
    for (int q = threadIdx.x; q < pz * px; q += BLOCK) {
      const int zz = q / px, xx = q - zz * px;
      const int gz = z0 + zz - hz, gx = x0 + xx - hx;
      T v = 0;
      if (gz >= 0 && gz < g.nz && gx >= 0 && gx < g.nx) {
        const int64_t pt = (int64_t)gz * g.nx + gx;
        v = usep ? r[pt] + beta * po[pt] : r[pt];
      }
      sp[q] = v;
    }
    __syncthreads();
    // G, row pass: h1[zz][xx] = sum_c K_x[c] p[zz][xx + c]  (xx over the S G p columns)
    for (int q = threadIdx.x; q < pz * sx; q += BLOCK) {
      const int zz = q / sx, xx = q - zz * sx;
      T a = 0;
      for (int c = 0; c < g.kw; ++c) a += (T)P.gx[c] * sp[zz * px + xx + c];
      h1[q] = a;
    }
    __syncthreads();
    // G, column pass, then the mask S (0 outside the grid)
    for (int q = threadIdx.x; q < sz * sx; q += BLOCK) {
      const int zz = q / sx, xx = q - zz * sx;
      const int gz = z0 + zz - rz, gx = x0 + xx - rx;
      T a = 0;
      if (gz >= 0 && gz < g.nz && gx >= 0 && gx < g.nx && g.mask[(int64_t)gz * g.nx + gx]) {
        for (int rr = 0; rr < g.kh; ++rr) a += (T)P.gz_[rr] * h1[(zz + rr) * sx + xx];
      }
      ss[q] = a;
    }
    __syncthreads();
    // G^T = the mirrored taps: row pass, then column pass on the interior
    for (int q = threadIdx.x; q < sz * BF_TX; q += BLOCK) {
      const int zz = q / BF_TX, xx = q - zz * BF_TX;
      T a = 0;
      for (int c = 0; c < g.kw; ++c) a += (T)P.gx[g.kw - 1 - c] * ss[zz * sx + xx + c];
      h2[q] = a;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < BF_TZ * BF_TX; q += BLOCK) {
      const int zz = q / BF_TX, xx = q - zz * BF_TX;
      const int gz = z0 + zz, gx = x0 + xx;
      if (gz >= g.nz || gx >= g.nx) continue;
      T a = 0;
      for (int rr = 0; rr < g.kh; ++rr) a += (T)P.gz_[g.kh - 1 - rr] * h2[(zz + rr) * BF_TX + xx];
      P.ub[(int64_t)gz * g.nx + gx] = cF * a;
    }
    __syncthreads();
  }
}

}  // namespace sip
