// sip_aux_kernels.cuh -- layout marshalling and multilevel transfer kernels.
//   k_pack / k_unpack : padded grid-shaped field block <-> compact paper layout
//   k_apply_op        : s = A_i x for the step-level entry point sip_apply_op
//   k_apply_sys       : q = C p for sip_apply_system / sip_cg's r = b - C x
//   k_restrict        : 2x2(x2) block mean + stride 2 (reading L23)
//   k_prolong         : (tri)linear align-corners interpolation of a field as an
//                       image of its own shape (reading L23)
#pragma once
#include "sip_kernels.cuh"

namespace sip {

// compact index of padded entry (prim, pt) inside its block, or -1 on pads
__device__ __forceinline__ long long compact_index(const Geo& g, int prim, const Loc& L, int pt,
                                                   const int* fmap) {
  switch (prim) {
    case PRIM_I: return pt;
    case PRIM_Z: return (L.gz < g.nz_g - 1) ? (long long)pt : -1;
    case PRIM_Y: return (L.iy < g.ny - 1) ? ((long long)L.iz * (g.ny - 1) + L.iy) * g.nx + L.ix : -1;
    case PRIM_X: return (L.ix < g.nx - 1) ? ((long long)L.iz * g.ny + L.iy) * (g.nx - 1) + L.ix : -1;
    default: return fmap[pt];
  }
}

// dir 0: padded -> compact (out[boff + ci] = field[b*ld + pt]); dir 1: compact -> padded
template <class T, class U>
__global__ void k_pack(Geo g, int prim, const int* fmap, long long boff, T* field, U* comp, int dir) {
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < g.N; pt += gridDim.x * blockDim.x) {
    Loc L = locate(g, pt);
    long long ci = compact_index(g, prim, L, pt, fmap);
    if (dir == 0) {
      if (ci >= 0) comp[boff + ci] = (U)field[pt];
    } else {
      field[pt] = (ci >= 0) ? (T)comp[boff + ci] : (T)0;
    }
  }
}

template <class T>
__global__ void k_apply_op(const __grid_constant__ Prob<T> P, int set_id, const T* x, T* out) {
  const Geo& g = P.g;
  const SetD<T>& S = P.set[set_id];
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < g.N; pt += gridDim.x * blockDim.x) {
    Loc L = locate(g, pt);
    for (int b = 0; b < S.nblk; ++b) {
      const int prim = S.prim[b];
      double s = is_pad(g, prim, L, pt) ? 0.0 : prim_fwd(g, P.taps, prim, VF<T>{x}, pt, L);
      out[(int64_t)b * g.ld + pt] = (T)s;
    }
  }
}

// mode 0: q = C p; mode 1: q = b - C p (initial CG residual)
template <class T>
__global__ void k_apply_sys(const __grid_constant__ Prob<T> P, const Ctrl* Cc, const T* p, const T* b,
                            T* q, int mode) {
  const Geo& g = P.g;
  const Ctrl& C = *Cc;
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < g.N; pt += gridDim.x * blockDim.x) {
    Loc L = locate(g, pt);
    double v = apply_C_at(P, C, VF<T>{p}, pt, L);
    q[pt] = (T)(mode == 0 ? v : (double)b[pt] - v);
  }
}

// "anti-alias filtering and subsampling", reading L23: every coarse
// point is the mean of its 2 x 2 (x 2) fine block.  The block is summed as x
// pairs, then y, then z (a pairwise tree); one multiply by 1/4 (1/8).
template <class T>
__global__ void k_restrict(Geo fine, Geo coarse, const T* f, T* c) {
  const bool three = fine.ndim == 3;
  const double scale = three ? 0.125 : 0.25;
  const int64_t fplane = (int64_t)fine.ny * fine.nx;
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < coarse.N; pt += gridDim.x * blockDim.x) {
    const Loc L = locate(coarse, pt);
    const T* q = f + (int64_t)(2 * L.iz) * fplane + (int64_t)(three ? 2 * L.iy : L.iy) * fine.nx + 2 * L.ix;
    auto row = [&](const T* r) { return (double)r[0] + (double)r[1]; };
    auto plane = [&](const T* r) { return three ? row(r) + row(r + fine.nx) : row(r); };
    c[pt] = (T)((plane(q) + plane(q + fplane)) * scale);
  }
}

// align-corners linear weights on one axis (reading L23): fine index i of nf
// sits at i (nc - 1) / (nf - 1) on the coarse axis; the integer part and the
// remainder are taken exactly in integer arithmetic
struct AxisW {
  int a, b;      // the two coarse neighbours
  double t;      // weight of b
};
__device__ __forceinline__ AxisW axis_weights(int i, int nf, int nc) {
  AxisW w{0, 0, 0.0};
  if (nf <= 1 || nc <= 1) return w;
  const long long num = (long long)i * (nc - 1);
  w.a = (int)(num / (nf - 1));
  const long long rem = num - (long long)w.a * (nf - 1);
  w.t = (double)rem / (double)(nf - 1);
  w.b = w.a + 1 < nc ? w.a + 1 : w.a;
  return w;
}
__device__ __forceinline__ double lerp1(double u, double v, double t) { return u + t * (v - u); }

// prolong one block of a field.  The block's real entries form an image of
// shape (ez, ey, ex) = grid shape minus 1 along the primitive's axis; it is
// interpolated from the coarse image of the same kind.  Pads are set to 0.
//
// z slabs: z is mapped in global plane numbers (nz_g, z0 of each level); the
// coarse planes a fine slab needs lie within one plane of the coarse slab
// (the coarse field's ghost planes, filled by the runtime's halo exchange).
template <class T>
__global__ void k_prolong(Geo fine, Geo coarse, int prim, const T* c, T* f) {
  const int dz = prim == PRIM_Z, dy = prim == PRIM_Y, dx = prim == PRIM_X;
  const int cz = coarse.nz_g - dz, cy = coarse.ny - dy, cx = coarse.nx - dx;
  const int fz = fine.nz_g - dz, fy = fine.ny - dy, fx = fine.nx - dx;
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < fine.N; pt += gridDim.x * blockDim.x) {
    Loc L = locate(fine, pt);
    if (L.gz >= fz || L.iy >= fy || L.ix >= fx) { f[pt] = (T)0; continue; }
    const AxisW wz = axis_weights(L.gz, fz, cz), wy = axis_weights(L.iy, fy, cy), wx = axis_weights(L.ix, fx, cx);
    const int za = wz.a - coarse.z0, zb = wz.b - coarse.z0;   // local coarse planes, -1 .. coarse.nz (ghosts)
    auto at = [&](int z, int y, int x) { return (double)c[((int64_t)z * coarse.ny + y) * coarse.nx + x]; };
    auto along_x = [&](int z, int y) { return lerp1(at(z, y, wx.a), at(z, y, wx.b), wx.t); };
    auto along_y = [&](int z) { return lerp1(along_x(z, wy.a), along_x(z, wy.b), wy.t); };
    f[pt] = (T)lerp1(along_y(za), along_y(zb), wz.t);
  }
}

// relative radius of a transform-domain l1 set: sigma = frac ||D m||_1
// (reading L30); c holds D m.  Fixed-order reduction (partials, last CTA).
template <class T>
__global__ void __launch_bounds__(BLOCK) k_dct_sigma(const __grid_constant__ Prob<T> P, int i, const T* c) {
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  double a = 0.0;
  for (long long q = blockIdx.x * (long long)BLOCK + threadIdx.x; q < P.g.N; q += (long long)gridDim.x * BLOCK)
    a += fabs((double)c[q]);
  a = block_sum(a, sh);
  if (threadIdx.x == 0) P.partials[blockIdx.x] = a;
  if (last_block(P.counter)) {
    reduce_partials(P.partials, 1, out, sh);
    if (threadIdx.x == 0) {
      *P.counter = 0u;
      Ctrl& C = *P.ctrl;
      C.sigma[i] = C.u_sigma[i] * out[0];
      for (int jb = 0; jb < C.njobs; ++jb)
        if (C.job[jb].set == i) C.job[jb].sigma = C.sigma[i];
    }
  }
}

// ---- Algorithm 4 (parallel Dykstra) vector steps
template <class T>
struct DykPtrs {
  T* y[MAXP];
  T* v[MAXP];
};
// x_old = x; x = sum_i y_i / p (step 2); v_i = x + v_i - y_i (step 3);
// out = (||x - x_old||^2, ||x||^2), fixed-order reduction
template <class T>
__global__ void __launch_bounds__(BLOCK) k_dyk_update(T* x, T* xo, DykPtrs<T> P, int p, long long n,
                                                      double* partials, unsigned* counter, double* out) {
  __shared__ double sh[NWARP + 1];
  __shared__ double o2[2];
  double d2 = 0.0, x2 = 0.0;
  const double w = 1.0 / (double)p;
  for (long long q = blockIdx.x * (long long)BLOCK + threadIdx.x; q < n; q += (long long)gridDim.x * BLOCK) {
    double a = 0.0;
    for (int i = 0; i < p; ++i) a += w * (double)P.y[i][q];
    const T xn = (T)a;
    const double d = (double)xn - (double)x[q];
    d2 += d * d;
    x2 += (double)xn * (double)xn;
    xo[q] = x[q];
    x[q] = xn;
    for (int i = 0; i < p; ++i) P.v[i][q] = xn + P.v[i][q] - P.y[i][q];
  }
  d2 = block_sum(d2, sh);
  x2 = block_sum(x2, sh);
  if (threadIdx.x == 0) { partials[blockIdx.x * 2] = d2; partials[blockIdx.x * 2 + 1] = x2; }
  if (last_block(counter)) {
    reduce_partials(partials, 2, o2, sh);
    if (threadIdx.x == 0) { *counter = 0u; out[0] = o2[0]; out[1] = o2[1]; }
  }
}
// (||a - pa||^2, ||a||^2) for Eq. 26
template <class T>
__global__ void __launch_bounds__(BLOCK) k_feas2(const T* a, const T* pa, long long n, double* partials,
                                                 unsigned* counter, double* out) {
  __shared__ double sh[NWARP + 1];
  __shared__ double o2[2];
  double d2 = 0.0, a2 = 0.0;
  for (long long q = blockIdx.x * (long long)BLOCK + threadIdx.x; q < n; q += (long long)gridDim.x * BLOCK) {
    const double d = (double)a[q] - (double)pa[q];
    d2 += d * d;
    a2 += (double)a[q] * (double)a[q];
  }
  d2 = block_sum(d2, sh);
  a2 = block_sum(a2, sh);
  if (threadIdx.x == 0) { partials[blockIdx.x * 2] = d2; partials[blockIdx.x * 2 + 1] = a2; }
  if (last_block(counter)) {
    reduce_partials(partials, 2, o2, sh);
    if (threadIdx.x == 0) { *counter = 0u; out[0] = o2[0]; out[1] = o2[1]; }
  }
}

template <class T>
__global__ void k_copy(const T* a, T* b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <class T>
__global__ void k_fill(T* a, long long n, T v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    a[i] = v;
}

}  // namespace sip
