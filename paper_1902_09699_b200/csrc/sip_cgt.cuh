// sip_cgt.cuh -- tile-staged flat CG kernels (sm_100a).
//
// The lean flat kernels (k_cg1f / k_cg2f, sip_vec.cuh) issue ~110 SASS
// instructions per warp-chunk but stall on their 7-10 dependent global loads
// (long scoreboard, ~3 TB/s).  Here each CTA owns one contiguous chunk range
// and streams it in tiles of BLOCK chunks; for every tile one thread issues
// 1D bulk copies (cp.async.bulk) of the operand's extended tile [start -
// (nx + W), end + nx + W) (x and y neighbours), its tiles one plane below and
// above (z neighbours) and the other streamed array, double-buffered on two
// mbarriers.  The stencil then reads shared memory only; the copies of the
// next tile are in flight meanwhile.  Arithmetic per point is that of the
// lean kernels (diagonal form, CGLoc).
#pragma once
#include "sip_stage.cuh"
#include "sip_vec.cuh"

namespace sip {

// elements of one staged copy of an operand (extended tile + two plane tiles)
template <class T>
__host__ __device__ inline int cgt_ext(int nx, bool hy) { return (hy ? nx : 0) + VT<T>::W; }
template <class T>
__host__ __device__ inline int cgt_opnd(int nx, bool hy) {
  const int n = BLOCK * VT<T>::W;
  return (n + 2 * cgt_ext<T>(nx, hy) + 2 * n + 31) / 32 * 32;
}
// dynamic shared memory of k_cg1t (two operands) / k_cg2t (operand + r tile), two stages
template <class T>
__host__ inline size_t cgt_smem(int nx, bool hy, bool cg1) {
  const int n = BLOCK * VT<T>::W;
  return (size_t)2 * (cg1 ? 2 * cgt_opnd<T>(nx, hy) : cgt_opnd<T>(nx, hy) + n) * sizeof(T);
}

// bulk copies of one operand's tile: [E | ZM | ZP] at dst
template <class T>
__device__ __forceinline__ unsigned cgt_issue_opnd(const Geo& g, const T* src, int64_t o, int np, int ext, T* dst,
                                                   uint64_t* bar) {
  const int n = BLOCK * VT<T>::W;
  const unsigned be = (unsigned)((np + 2 * ext) * sizeof(T)), bp = (unsigned)(np * sizeof(T));
  bulk_g2s(dst, src + o - ext, be, bar);
  bulk_g2s(dst + n + 2 * ext, src + o - g.plane, bp, bar);
  bulk_g2s(dst + 2 * n + 2 * ext, src + o + g.plane, bp, bar);
  return be + 2 * bp;
}

// the 7 neighbours of my chunk from a staged operand (optionally p = a + beta b)
template <class T, bool HY>
struct Nb7 {
  static constexpr int W = VT<T>::W;
  T cur[W], zm[W], zp[W], ym[W], yp[W], xl, xr;
  __device__ __forceinline__ void load(const T* s, int tid, int ext, int nx) {
    const int n = BLOCK * W;
    const int eb = ext + tid * W;
    VT<T>::ldT_s(s + eb, cur);
    xl = s[eb - 1];
    xr = s[eb + W];
    if (HY) {
      VT<T>::ldT_s(s + eb - nx, ym);
      VT<T>::ldT_s(s + eb + nx, yp);
    }
    VT<T>::ldT_s(s + n + 2 * ext + tid * W, zm);
    VT<T>::ldT_s(s + 2 * n + 2 * ext + tid * W, zp);
  }
  __device__ __forceinline__ void axpy(const Nb7& b, T beta) {   // this = this + beta b
#pragma unroll
    for (int e = 0; e < W; ++e) {
      cur[e] = cur[e] + beta * b.cur[e];
      zm[e] = zm[e] + beta * b.zm[e];
      zp[e] = zp[e] + beta * b.zp[e];
      if (HY) { ym[e] = ym[e] + beta * b.ym[e]; yp[e] = yp[e] + beta * b.yp[e]; }
    }
    xl = xl + beta * b.xl;
    xr = xr + beta * b.xr;
  }
};

template <class T, bool HY>
__global__ void __launch_bounds__(BLOCK, 3) k_cg1t(const __grid_constant__ Prob<T> P, int j) {
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
  extern __shared__ __align__(128) unsigned char sm_[];
  __shared__ uint64_t bar[2];
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  T* sb = reinterpret_cast<T*>(sm_);
  const int ext = cgt_ext<T>(g.nx, HY), op = cgt_opnd<T>(g.nx, HY);
  const bool usep = j > 0;
  const CoefT<T> k = coefs_present(P, C);
  const T beta = (T)C.beta;
  const T* po = usep ? p_slot(P, j - 1) : nullptr;
  T* pw = p_slot(P, j);
  const int ncr = g.nx / W;
  FastDiv dncr;
  dncr.d = P.dncr.d; dncr.m = P.dncr.m; dncr.l = P.dncr.l;
  const int per = (nch + (int)gridDim.x - 1) / (int)gridDim.x;
  const int c0 = min(nch, (int)blockIdx.x * per), c1 = min(nch, c0 + per);
  const int ntile = (c1 - c0 + BLOCK - 1) / BLOCK;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_fence_init(); }
  __syncthreads();
  unsigned ph = 0;
  auto issue = [&](int t) {
    if (threadIdx.x == 0) {
      const int s = t & 1;
      const int cs = c0 + t * BLOCK;
      const int np = min(BLOCK, c1 - cs) * W;
      const int64_t o = (int64_t)cs * W;
      const unsigned bytes = (unsigned)(((np + 2 * ext) + 2 * np) * sizeof(T));
      mbar_expect_tx(&bar[s], usep ? 2 * bytes : bytes);
      T* d = sb + (size_t)s * 2 * op;
      cgt_issue_opnd<T>(g, P.r, o, np, ext, d, &bar[s]);
      if (usep) cgt_issue_opnd<T>(g, po, o, np, ext, d + op, &bar[s]);
    }
  };
  double pq = 0.0;
  if (ntile > 0) issue(0);
  for (int t = 0; t < ntile; ++t) {
    if (t + 1 < ntile) issue(t + 1);
    const int s = t & 1;
    mbar_wait(&bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
    const int c = c0 + t * BLOCK + (int)threadIdx.x;
    if (c < c1) {
      const T* d = sb + (size_t)s * 2 * op;
      Nb7<T, HY> a;
      a.load(d, threadIdx.x, ext, g.nx);
      if (usep) {
        Nb7<T, HY> b;
        b.load(d + op, threadIdx.x, ext, g.nx);
        a.axpy(b, beta);
      }
      const CGLoc<T> L(g, k, c, ncr, dncr);
      T q[W];
      L.template apply<W>(a.cur, a.zm, a.zp, a.ym, a.yp, a.xl, a.xr, HY, q);
      VT<T>::stT(pw + c * W, a.cur);
      T sm = 0;
#pragma unroll
      for (int e = 0; e < W; ++e) sm += a.cur[e] * q[e];
      pq += (double)sm;
    }
    __syncthreads();   // stage s is refilled by the issue of tile t + 2
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

template <class T, bool HY>
__global__ void __launch_bounds__(BLOCK, 4) k_cg2t(const __grid_constant__ Prob<T> P, int j) {
  constexpr int W = VT<T>::W;
  Ctrl& C = *P.ctrl;
  if (C.stopped || !C.cg_active) return;
  extern __shared__ __align__(128) unsigned char sm_[];
  __shared__ uint64_t bar[2];
  __shared__ double sh[NWARP + 1];
  __shared__ double out[1];
  T* sb = reinterpret_cast<T*>(sm_);
  const Geo& g = P.g;
  const int nch = g.N / W;
  const int n = BLOCK * W;
  const int ext = cgt_ext<T>(g.nx, HY), op = cgt_opnd<T>(g.nx, HY);
  const int st_ = op + n;
  const CoefT<T> k = coefs_present(P, C);
  const T alpha = (T)C.alpha;
  const T* p = p_slot(P, j);
  const int ncr = g.nx / W;
  FastDiv dncr;
  dncr.d = P.dncr.d; dncr.m = P.dncr.m; dncr.l = P.dncr.l;
  const int per = (nch + (int)gridDim.x - 1) / (int)gridDim.x;
  const int c0 = min(nch, (int)blockIdx.x * per), c1 = min(nch, c0 + per);
  const int ntile = (c1 - c0 + BLOCK - 1) / BLOCK;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); mbar_fence_init(); }
  __syncthreads();
  unsigned ph = 0;
  auto issue = [&](int t) {
    if (threadIdx.x == 0) {
      const int s = t & 1;
      const int cs = c0 + t * BLOCK;
      const int np = min(BLOCK, c1 - cs) * W;
      const int64_t o = (int64_t)cs * W;
      mbar_expect_tx(&bar[s], (unsigned)((np + 2 * ext + 2 * np + np) * sizeof(T)));
      T* d = sb + (size_t)s * st_;
      cgt_issue_opnd<T>(g, p, o, np, ext, d, &bar[s]);
      bulk_g2s(d + op, P.r + o, (unsigned)(np * sizeof(T)), &bar[s]);
    }
  };
  double rr = 0.0;
  if (ntile > 0) issue(0);
  for (int t = 0; t < ntile; ++t) {
    if (t + 1 < ntile) issue(t + 1);
    const int s = t & 1;
    mbar_wait(&bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
    const int c = c0 + t * BLOCK + (int)threadIdx.x;
    if (c < c1) {
      const T* d = sb + (size_t)s * st_;
      Nb7<T, HY> a;
      a.load(d, threadIdx.x, ext, g.nx);
      T rv[W];
      VT<T>::ldT_s(d + op + threadIdx.x * W, rv);
      const CGLoc<T> L(g, k, c, ncr, dncr);
      T q[W];
      L.template apply<W>(a.cur, a.zm, a.zp, a.ym, a.yp, a.xl, a.xr, HY, q);
      T sm = 0;
#pragma unroll
      for (int e = 0; e < W; ++e) {
        rv[e] = rv[e] - alpha * q[e];
        sm += rv[e] * rv[e];
      }
      VT<T>::stT(P.r + c * W, rv);
      rr += (double)sm;
    }
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

}  // namespace sip
