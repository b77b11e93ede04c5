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

// block mean of the fine grid (2 x 2 in 2D over (z, x), 2 x 2 x 2 in 3D)
template <class T>
__global__ void k_restrict(Geo fine, Geo coarse, const T* f, T* c) {
  const int by = fine.ndim == 3 ? 2 : 1;
  const double inv = 1.0 / (double)(4 * by);
  for (int pt = blockIdx.x * blockDim.x + threadIdx.x; pt < coarse.N; pt += gridDim.x * blockDim.x) {
    Loc L = locate(coarse, pt);
    double a = 0.0;
    for (int dz = 0; dz < 2; ++dz)
      for (int dy = 0; dy < by; ++dy)
        for (int dx = 0; dx < 2; ++dx)
          a += (double)f[((int64_t)(2 * L.iz + dz) * fine.ny + (by * L.iy + dy)) * fine.nx + 2 * L.ix + dx];
    c[pt] = (T)(a * inv);
  }
}

__device__ __forceinline__ void axis_w(int i, int nf, int nc, int* i0, int* i1, double* t) {
  double pos = (nf > 1 && nc > 1) ? (double)i * (double)(nc - 1) / (double)(nf - 1) : 0.0;
  int a = (int)floor(pos);
  if (a > nc - 1) a = nc - 1;
  *i0 = a;
  *i1 = (a + 1 < nc) ? a + 1 : a;
  *t = pos - (double)a;
}

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
    int z0, z1, y0, y1, x0, x1;
    double tz, ty, tx;
    axis_w(L.gz, fz, cz, &z0, &z1, &tz);
    axis_w(L.iy, fy, cy, &y0, &y1, &ty);
    axis_w(L.ix, fx, cx, &x0, &x1, &tx);
    z0 -= coarse.z0;   // local coarse plane, -1 .. coarse.nz (ghosts)
    z1 -= coarse.z0;
    auto C_ = [&](int a, int b, int d) {  // coarse padded storage
      return (double)c[((int64_t)a * coarse.ny + b) * coarse.nx + d];
    };
    const double v00 = C_(z0, y0, x0) * (1.0 - tx) + C_(z0, y0, x1) * tx;
    const double v01 = C_(z0, y1, x0) * (1.0 - tx) + C_(z0, y1, x1) * tx;
    const double v10 = C_(z1, y0, x0) * (1.0 - tx) + C_(z1, y0, x1) * tx;
    const double v11 = C_(z1, y1, x0) * (1.0 - tx) + C_(z1, y1, x1) * tx;
    const double v0 = v00 * (1.0 - ty) + v01 * ty;
    const double v1 = v10 * (1.0 - ty) + v11 * ty;
    f[pt] = (T)(v0 * (1.0 - tz) + v1 * tz);
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
