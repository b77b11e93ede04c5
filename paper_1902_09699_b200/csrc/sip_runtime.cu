// sip_runtime.cu -- host runtime and C ABI (include/sip.h) of the B200 PARSDMM
// hot path (arXiv 1902.09699).  One Engine<T> per grid level owns the device
// state; the iteration (Algorithm 1) is enqueued as a fixed kernel sequence
// whose decisions live in device memory (Ctrl), captured once into a CUDA
// graph of `graph_iters` iterations and replayed; the host reads one flag per
// graph launch (lagged by one launch) to learn that Eq. 28 stopped the run.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/sip.h"
#include "sip_aux_kernels.cuh"
#include "sip_team.cuh"
#include "sip_fiber.cuh"
#include "sip_svd.cuh"
#include "sip_blur.cuh"
#include "sip_select_small.cuh"

using namespace sip;

namespace {

struct SipError {
  sip_status code;
  std::string msg;
};

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw SipError{SIP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};   \
  } while (0)

struct HostSet {
  sip_op op;
  sip_set_type type;
  sip_set_params prm;
  std::vector<double> lo_vec, hi_vec;   // compact layout
  std::vector<double> kernel;
  int kh = 0, kw = 0;
  std::vector<uint8_t> mask;
  int64_t M = 0;
  int zero_in = 1;
  int fib = 0;          // 0 whole vector; 1 x-fibers; 2 z-fibers (app_mode)
  int64_t flen = 0;     // fiber length
};

struct Options {
  double rho0 = 1e-2, gamma0 = 1.0, eps_corr = 0.3, rho_ratio_cap = 1e3, gamma_max = 2.0 - 1e-3;
  int n_cg = 10, eq25 = 1, fixed_work = 0, adapt_every = 2, check_every = 5;
  double eps_evol = -1.0;       // < 0: 10 * tol
  double cg_tol_floor = -1.0;   // < 0: 10 * eps(dtype)
  int warm_start = 0, graph_iters = 10, profile = 0;
};

inline int nblk_of(sip_op op, int ndim) {
  return op == SIP_OP_TV ? (ndim == 3 ? 3 : 2) : 1;
}
inline void prims_of(sip_op op, int ndim, int* pr) {
  switch (op) {
    case SIP_OP_IDENTITY: pr[0] = PRIM_I; break;
    case SIP_OP_DZ: pr[0] = PRIM_Z; break;
    case SIP_OP_DY: pr[0] = PRIM_Y; break;
    case SIP_OP_DX: pr[0] = PRIM_X; break;
    case SIP_OP_TV:
      pr[0] = PRIM_Z;
      if (ndim == 3) { pr[1] = PRIM_Y; pr[2] = PRIM_X; } else { pr[1] = PRIM_X; }
      break;
    default: pr[0] = PRIM_F;
  }
}
inline int kind_of(sip_set_type t) {
  switch (t) {
    case SIP_SET_BOUNDS: return K_BOUNDS;
    case SIP_SET_L1_BALL: return K_L1;
    case SIP_SET_L2_BALL: return K_L2;
    case SIP_SET_ANNULUS: return K_ANN;
    case SIP_SET_RANK: return K_RANK;
    case SIP_SET_DCT_L1: return K_L1;
    case SIP_SET_HAAR_L1: return K_L1;
    case SIP_SET_NUCLEAR: return K_NUC;
    default: return K_CARD;
  }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ------------------------------------------------------------------ engine
struct EngineBase {
  virtual ~EngineBase() {}
};

template <class T>
struct Engine : EngineBase {
  // configuration
  int ndim;
  int nz, ny, nx;
  double h[3];
  cudaStream_t stream;
  int nsm = 148;
  int nfib_sets = 0;             // sets applied per fiber (k_fiber)
  int nsvd_sets = 0, g_svd = 0;  // rank / nuclear-norm sets (sip_svd.cuh): a cluster of svd_cl CTAs per matrix
  int svd_cl[SIP_MAX_SETS] = {};
  // orthogonal-transform l1 sets (NEXT-3): the orthonormal DCT-II
  // of the grid by cuBLAS GEMMs along each axis (plain library GEMMs)
  bool cgv = false;              // vectorised CG kernels (vec, or vec except a separable blur set)
  bool sel_small = false;        // every radix job small: k_selsmall (one CTA per job)
  bool selc_fused = false;       // select v2: the candidate rounds in one launch (k_selCF)
  size_t smem_bf = 0;
  int g_bf = 1;
  int ndct_sets = 0;
  cublasHandle_t blas = nullptr;
  T* dctm[2][3] = {};   // column-major transform matrices (DCT-II, Haar) of the z, y, x axes
  T* dtmp = nullptr;                           // one N-field of scratch
  void* blas_ws = nullptr;
  int g_fib = 0, g_fibw = 0, nfib_sort = 0, nfib_warp = 0;
  int g_fw[MAXP] = {0};
  size_t smem_fib = 0, smem_fw[MAXP] = {0};
  const std::vector<HostSet>* sets;
  int p, P;
  // device state
  Prob<T> Pr;
  std::vector<void*> allocs;
  Ctrl* d_ctrl = nullptr;
  Ctrl hc;
  int* d_fmap = nullptr;      // blur mask compact index map
  int* d_log_cg = nullptr; int* d_log_br = nullptr;
  double* d_log_rho = nullptr; double* d_log_gam = nullptr; double* d_log_feas = nullptr;
  double* d_log_evol = nullptr;
  unsigned long long* d_log_supp = nullptr;
  int log_cap = 0;
  int* h_flag = nullptr;       // pinned: stopped flags of the last launches
  cudaEvent_t ev_flag[2];
  cudaEvent_t ev0, ev1;
  // launch geometry
  int g_pts = 1, g_sel = 1, g_p2 = 1, g_small = 1, g_vec = 1, g_p1 = 1, g_p1a = 1;
  int npr = 0;                   // allocated slots of the p ring (Prob::pr)
  bool l2_window = false;        // an L2 persisting window on r (set on the stream before capture)
  cudaStreamAttrValue l2av;
  void apply_l2_window() {   // this engine's window, or none (the stream is shared by levels)
    cudaStreamAttrValue none;
    memset(&none, 0, sizeof(none));
    CU(cudaStreamSetAttribute(stream, cudaStreamAttributeAccessPolicyWindow, l2_window ? &l2av : &none));
  }
  int g_cg1p = 1, g_cg2p = 1, g_rhsp = 1;   // lean CG / rhs grids (z pairs)
  bool vec = false;
  size_t smem_p1 = 0, smem_p2 = 0, smem_init = 0, smem_p1v = 0, smem_p1a = 0;
  // graph
  cudaGraphExec_t gexec = nullptr;
  int g_iters = 0, g_ncg = -1;
  bool g_prof = false;
  int g_ce = 0;
  long long launches = 0;       // kernels enqueued by the last project()
  long long graph_kernels = 0;  // kernels in one captured graph
  int last_k = 0;               // Ctrl.k after the last run
  bool ran = false;
  bool scratch_used = false;    // state buffers overwritten by a step-level call

  ~Engine() override {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (blas) cublasDestroy(blas);
    for (void* a : allocs) cudaFree(a);
    if (h_flag) cudaFreeHost(h_flag);
    cudaEventDestroy(ev_flag[0]); cudaEventDestroy(ev_flag[1]);
    cudaEventDestroy(ev0); cudaEventDestroy(ev1);
  }

  template <class Q>
  Q* dalloc(size_t n) {
    void* p_ = nullptr;
    cudaError_t e = cudaMalloc(&p_, std::max<size_t>(n, 1) * sizeof(Q));
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw SipError{SIP_ERR_OOM, "cudaMalloc of " + std::to_string(n * sizeof(Q)) + " bytes failed"};
    }
    allocs.push_back(p_);
    return (Q*)p_;
  }

  // field of nblk blocks; returns pointer to block 0's first interior element
  // guard bands (SIP_CANARY=1, a bounds check of our own): every field gets
  // CANARY_N words before and after its storage filled with a canary pattern,
  // checked after each solve -- any kernel writing outside a field's
  // allocation (ghost planes included) is reported as SIP_ERR_CUDA
  static constexpr size_t CANARY_N = 4096;
  const bool canary = getenv("SIP_CANARY") != nullptr;
  std::vector<std::pair<T*, size_t>> guards;
  T* field(int nblk) {
    const size_t n = (size_t)nblk * Pr.g.ld;
    if (canary) {
      T* raw = dalloc<T>(n + 2 * CANARY_N);
      CU(cudaMemsetAsync(raw, 0xA5, CANARY_N * sizeof(T), stream));
      CU(cudaMemsetAsync(raw + CANARY_N, 0, n * sizeof(T), stream));
      CU(cudaMemsetAsync(raw + CANARY_N + n, 0xA5, CANARY_N * sizeof(T), stream));
      guards.push_back({raw, n});
      return raw + CANARY_N + (size_t)GHOST * Pr.g.plane;
    }
    T* base = dalloc<T>(n);
    CU(cudaMemsetAsync(base, 0, n * sizeof(T), stream));
    return base + (size_t)GHOST * Pr.g.plane;
  }
  void check_canaries() {
    if (!canary) return;
    std::vector<unsigned char> h(CANARY_N * sizeof(T));
    for (size_t f = 0; f < guards.size(); ++f) {
      for (int side = 0; side < 2; ++side) {
        const T* p = guards[f].first + (side ? CANARY_N + guards[f].second : 0);
        CU(cudaMemcpy(h.data(), p, h.size(), cudaMemcpyDeviceToHost));
        for (size_t b = 0; b < h.size(); ++b)
          if (h[b] != 0xA5)
            throw SipError{SIP_ERR_CUDA, "SIP_CANARY: write outside field " + std::to_string(f) +
                                             (side ? " (after its end)" : " (before its start)")};
      }
    }
  }

  // slab: this engine owns global planes [z0_, z0_ + nz_) of nz_g_ (rank of nranks_)
  int z0 = 0, nz_g = 0, nranks = 1, rank = 0;

  void setup(int ndim_, int nz_, int ny_, int nx_, const double* h_, cudaStream_t st,
             const std::vector<HostSet>& s, int z0_ = 0, int nz_g_ = -1, int nranks_ = 1, int rank_ = 0) {
    ndim = ndim_; nz = nz_; ny = ny_; nx = nx_;
    z0 = z0_; nz_g = nz_g_ < 0 ? nz_ : nz_g_; nranks = nranks_; rank = rank_;
    h[0] = h_[0]; h[1] = h_[1]; h[2] = h_[2];
    stream = st;
    sets = &s;
    p = (int)s.size();
    P = p + 1;
    int dev;
    CU(cudaGetDevice(&dev));
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    memset(&Pr, 0, sizeof(Pr));
    Geo& g = Pr.g;
    g.ndim = ndim; g.nz = nz; g.ny = ny; g.nx = nx; g.nz_g = nz_g; g.z0 = z0;
    g.plane = ny * nx;
    g.N = nz * g.plane;
    g.ld = (int64_t)g.N + 2 * GHOST * (int64_t)g.plane;
    g.ihz = 1.0 / h[0]; g.ihy = 1.0 / h[1]; g.ihx = 1.0 / h[2];
    g.dplane.init((uint32_t)g.plane);
    g.dnx.init((uint32_t)g.nx);
    g.dny.init((uint32_t)g.ny);
    Pr.dncr.init((uint32_t)std::max(1, g.nx / VT<T>::W));
    Pr.P = P; Pr.p = p;
    Pr.nranks = nranks; Pr.rank = rank;
    pdl = nranks == 1 && getenv("SIP_PDL");   // measured: no gain on the radix path, -4% to -20% with select v2 (early-launched CTAs hold SM resources)
    Pr.rounds = KeyT<T>::ROUNDS;
    Pr.ntiles_pb = (g.N + BLOCK - 1) / BLOCK;
    Pr.nseg1 = 0;   // counts (set, block) segments below; +1 for the x segment after
    int njobs = 0;
    for (int i = 0; i < P; ++i) {
      SetD<T>& S = Pr.set[i];
      if (i == p) {
        S.kind = K_DIST; S.nblk = 1; S.prim[0] = PRIM_I;
      } else {
        const HostSet& hs = s[i];
        S.kind = kind_of(hs.type);
        S.nblk = nblk_of(hs.op, ndim);
        prims_of(hs.op, ndim, S.prim);
        S.lo = hs.prm.lo; S.hi = hs.prm.hi;
        if (hs.op == SIP_OP_BLUR_MASK) {
          g.kh = hs.kh; g.kw = hs.kw;
          for (int t = 0; t < hs.kh * hs.kw; ++t) Pr.taps[t] = hs.kernel[t];
        }
      }
      S.global = (S.kind == K_L1 || S.kind == K_L2 || S.kind == K_ANN || S.kind == K_CARD ||
                  S.kind == K_RANK || S.kind == K_NUC);
      S.svd = (S.kind == K_RANK || S.kind == K_NUC);
      if (S.svd) nsvd_sets++;
      S.dct = i >= p ? 0 : s[i].type == SIP_SET_DCT_L1 ? 1 : s[i].type == SIP_SET_HAAR_L1 ? 2 : 0;
      if (S.dct) ndct_sets++;
      S.job = S.sjob = -1;
      S.fib = (i < p) ? s[i].fib : 0;
      // fiber length on this engine's own grid (multilevel levels differ)
      S.flen = !S.fib ? 0 : S.fib == 1 ? g.nx - (S.prim[0] == PRIM_X ? 1 : 0)
                                       : nz_g - (S.prim[0] == PRIM_Z ? 1 : 0);
      if ((S.kind == K_L1 || S.kind == K_CARD) && !S.fib) { S.job = njobs++; S.sjob = njobs++; }
      if (S.fib) nfib_sets++;
      // warp kernel for fibers of <= 32 FW_E entries (z-fibers: tiles that
      // fit in shared memory); SIP_FIBER_SORT=1 keeps the sort kernel (A/B)
      S.fpath = S.fib && S.flen <= 32 * FW_E && !getenv("SIP_FIBER_SORT") &&
                (S.fib == 1 || fiberw_smem(S.flen, (int)sizeof(T)) <= 200 * 1024);
      for (int b = 0; b < S.nblk; ++b) Pr.has[S.prim[b]] = 1;
      if (S.global) Pr.nglob++;
      for (int b = 0; b < S.nblk; ++b) {
        Pr.seg_set[1 + Pr.nseg1] = (short)i; Pr.seg_blk[1 + Pr.nseg1] = (short)b; Pr.nseg1++;
        if (S.global && !S.fib && !S.svd) { Pr.seg2_set[Pr.nseg2] = (short)i; Pr.seg2_blk[Pr.nseg2] = (short)b; Pr.nseg2++; }
      }
    }
    Pr.nseg1 += 1;   // segment 0: the per-point x work
    if (z0 > 0)
      for (int i = 0; i < P; ++i) Pr.set[i].first_real = -1;   // global index 0 is on rank 0 (L7)
    // blur mask + compact map
    for (int i = 0; i < p; ++i)
      if (s[i].op == SIP_OP_BLUR_MASK) {
        uint8_t* dm = dalloc<uint8_t>(g.N);
        CU(cudaMemcpyAsync(dm, s[i].mask.data(), g.N, cudaMemcpyHostToDevice, stream));
        g.mask = dm;
        std::vector<int> fm(g.N);
        int c = 0;
        for (int q = 0; q < g.N; ++q) fm[q] = s[i].mask[q] ? c++ : -1;
        d_fmap = dalloc<int>(g.N);
        CU(cudaMemcpyAsync(d_fmap, fm.data(), g.N * sizeof(int), cudaMemcpyHostToDevice, stream));
        CU(cudaStreamSynchronize(stream));
        Pr.set[i].first_real = 0;
        for (int q = 0; q < g.N; ++q) if (s[i].mask[q]) { Pr.set[i].first_real = q; break; }
      }
    // fields
    for (int i = 0; i < P; ++i) {
      SetD<T>& S = Pr.set[i];
      S.y[0] = field(S.nblk); S.y[1] = field(S.nblk);
      S.v[0] = field(S.nblk); S.v[1] = field(S.nblk);
      S.vh0 = field(S.nblk);
      S.w = S.global ? field(S.nblk) : nullptr;
      S.s = (S.kind == K_L1 || S.kind == K_CARD || S.svd) ? field(S.nblk) : nullptr;
      if (i < p && (!s[i].lo_vec.empty() || !s[i].hi_vec.empty())) {
        if (!s[i].lo_vec.empty()) S.lo_vec = upload_compact(i, s[i].lo_vec);
        if (!s[i].hi_vec.empty()) S.hi_vec = upload_compact(i, s[i].hi_vec);
      }
    }
    Pr.x = field(1);
    Pr.m = field(1);
    Pr.r = field(1);
    // keep the CG residual r resident in L2 (persisting access window on the
    // work stream): every CG step reads it (k_cg1 stencil) and reads + writes
    // it (k_cg2); with r in L2 a step moves ~4N words from DRAM instead of 6N.
    // The window is captured into the iteration graph's kernel nodes.
    // Only when r fits in a third of L2 (C4: 33.5 MB of 126 MB): a larger
    // carve-out starves every other kernel (measured on C5-L1, r = 268 MB:
    // all kernels ~2x slower).
    if (!getenv("SIP_NO_L2_PERSIST")) {
      int maxp = 0, maxw = 0, l2 = 0, dev = 0;
      CU(cudaGetDevice(&dev));
      CU(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
      CU(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev));
      CU(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
      const size_t rb = (size_t)g.ld * sizeof(T);
      if (maxp > 0 && maxw > 0 && rb <= (size_t)l2 / 3 && rb <= (size_t)maxp && rb <= (size_t)maxw) {
        size_t cur = 0;
        CU(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
        const size_t want = std::min((size_t)maxp, rb);
        if (cur < want) CU(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
        cudaStreamAttrValue av;
        memset(&av, 0, sizeof(av));
        av.accessPolicyWindow.base_ptr = (void*)(Pr.r - (size_t)GHOST * g.plane);
        av.accessPolicyWindow.num_bytes = std::min(rb, (size_t)maxw);
        av.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)want / (double)av.accessPolicyWindow.num_bytes);
        av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        l2av = av;
        l2_window = true;
      }
    }
    Pr.pb[0] = field(1); Pr.pb[1] = field(1);
    Pr.pr[0] = Pr.pb[0]; Pr.pr[1] = Pr.pb[1];
    npr = 2;
    Pr.defer_x = 0;
    Pr.tb = Pr.has[PRIM_F] ? field(1) : nullptr;
    for (int j = 0; j < HIST_S; ++j) Pr.hist[j] = field(1);
    Pr.xs[0] = field(1); Pr.xs[1] = field(1);
    // launch geometry
    const int tiles = Pr.ntiles_pb;
    g_pts = std::max(1, std::min(tiles, nsm * 8));
    g_sel = std::max(1, std::min(tiles, nsm * 4));
    g_p2 = std::max(1, std::min(tiles * 3, nsm * 8));
    g_small = std::max(1, std::min(tiles, nsm * 4));
    // vectorised CG kernels: W = 16/sizeof(T) points per thread along x
    constexpr int W = VT<T>::W;
    vec = (g.nx % W == 0) && !Pr.has[PRIM_F] && !getenv("SIP_NO_VEC");
    // the vectorised CG kernels also serve a grid with the blur / mask
    // operator when its kernel is separable (K = g_z g_x^T): the operator's
    // term of C p comes from k_blurF (sip_blur.cuh); the set passes stay scalar
    cgv = vec;
    if (Pr.has[PRIM_F] && (g.nx % W == 0) && !getenv("SIP_NO_VEC") && !getenv("SIP_BLUR_SCALAR") && nranks == 1) {
      for (int i = 0; i < p; ++i) {
        if (s[i].op != SIP_OP_BLUR_MASK) continue;
        const int kh = s[i].kh, kw = s[i].kw;
        const std::vector<double>& K = s[i].kernel;
        int r0 = 0, c0 = 0;
        for (int a = 0; a < kh * kw; ++a) if (std::fabs(K[a]) > std::fabs(K[r0 * kw + c0])) { r0 = a / kw; c0 = a % kw; }
        const double piv = K[r0 * kw + c0];
        double kmax = std::fabs(piv), err = 0.0;
        for (int rr = 0; rr < kh; ++rr) Pr.gz_[rr] = K[rr * kw + c0];
        for (int cc = 0; cc < kw; ++cc) Pr.gx[cc] = piv != 0.0 ? K[r0 * kw + cc] / piv : 0.0;
        for (int rr = 0; rr < kh; ++rr)
          for (int cc = 0; cc < kw; ++cc) err = std::max(err, std::fabs(K[rr * kw + cc] - Pr.gz_[rr] * Pr.gx[cc]));
        if (piv != 0.0 && err <= 1e-12 * kmax) {
          cgv = true;
          smem_bf = blurf_smem(kh, kw, sizeof(T));
          CU(cudaFuncSetAttribute(k_blurF<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bf));
          int occ = 0;
          CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_blurF<T>, BLOCK, smem_bf));
          const int tiles = ((g.nx + BF_TX - 1) / BF_TX) * ((g.nz + BF_TZ - 1) / BF_TZ);
          g_bf = std::max(1, std::min(tiles, nsm * std::max(occ, 1)));
        }
      }
    }
    if (nfib_sets && !vec)
      throw SipError{SIP_ERR_CONFIG, "per-fiber sets need nx % (16 / sizeof(dtype)) == 0 and no blur/mask operator"};
    if (ndct_sets && (!vec || nranks > 1))
      throw SipError{SIP_ERR_CONFIG, "transform-domain l1 sets need nx % (16 / sizeof(dtype)) == 0, no blur/mask operator, one rank"};
    if (ndct_sets) setup_dct();
    if (nsvd_sets && (!vec || nranks > 1))
      throw SipError{SIP_ERR_CONFIG, "rank / nuclear sets need nx % (16 / sizeof(dtype)) == 0, no blur/mask operator, one rank"};
    if (nsvd_sets) {   // fp64 scratch of the batched Jacobi kernel: X (m x n) and V (n x n) per matrix
      size_t nx_ = 0, nv_ = 0;
      for (int i = 0; i < p; ++i) {
        if (!Pr.set[i].svd) continue;
        const MatView mv = mat_view(ndim, nz_g, ny, nx, Pr.set[i].prim[0]);
        nx_ = std::max(nx_, (size_t)mv.nmat * mv.m * mv.n);
        nv_ = std::max(nv_, (size_t)mv.nmat * mv.n * mv.n);
        // few large matrices: a cluster of CTAs per matrix (the column
        // pairs of a round split over the cluster, sip_svd.cuh)
        int cl = 1;
        if (!getenv("SIP_SVD_CL1") && mv.n >= 64)
          for (int c : {16, 8, 4}) {
            if (mv.nmat * c > 2 * nsm) continue;
            if (c > 8) CU(cudaFuncSetAttribute(k_svdproj<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(mv.nmat * c));
            cfg.blockDim = dim3((unsigned)SVD_BLOCK);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = (unsigned)c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, k_svdproj<T>, &cfg) == cudaSuccess && ncl > 0) { cl = c; break; }
            cudaGetLastError();
          }
        svd_cl[i] = cl;
        g_svd = std::max(g_svd, mv.nmat * cl);
      }
      Pr.svdX = dalloc<double>(nx_);
      Pr.svdV = dalloc<double>(nv_);
    }
    g_vec = std::max(1, std::min((g.N / W + BLOCK - 1) / BLOCK, nsm * 8));
    // lean CG / rhs: one wave of resident CTAs (4 per SM)
    // CG over z pairs (one thread, two chunks): one resident wave, 4 (k_cg1f)
    // / 3 (k_cg2f, 77 registers) CTAs per SM, fewer if the registers say so
    auto wave = [&](const void* fn, int want) {
      int occ = 0;
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, BLOCK, 0));
      return std::max(1, std::min((g.N / W / 2 + BLOCK - 1) / BLOCK, nsm * std::max(1, std::min(occ, want))));
    };
    g_cg1p = wave(ndim == 3 ? (const void*)k_cg1f<T, true> : (const void*)k_cg1f<T, false>, 4);
    g_cg2p = wave(ndim == 3 ? (const void*)k_cg2f<T, true> : (const void*)k_cg2f<T, false>, CG2_MINB);
    g_rhsp = wave(ndim == 3 ? (const void*)k_rhsp<T, true> : (const void*)k_rhsp<T, false>, 3);
    const int nv1 = P * NSLOT + NEVOL;
    smem_p1 = (size_t)NWARP * nv1 * sizeof(double);   // scalar k_pass1
    // select v2 (sip_select2.cuh): single-rank fp32 runs with a radix job
    // (transform-domain sets: pass 1's round A would count untransformed keys)
    // small jobs (every radix job <= SEL_SMALL_MAX entries, one rank): one
    // sorting CTA per job (sip_select_small.cuh)
    sel_small = nranks == 1 && njobs > 0 && !getenv("SIP_SEL_V1");
    for (int i = 0; i < P && sel_small; ++i)
      if (Pr.set[i].job >= 0 && (long long)Pr.set[i].nblk * g.N > SEL_SMALL_MAX) sel_small = false;
    if (sel_small) CU(cudaFuncSetAttribute(k_selsmall<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)selsmall_smem()));
    Pr.selv2 = (vec && sizeof(T) == 4 && nranks == 1 && njobs > 0 && !ndct_sets && !sel_small && !getenv("SIP_SEL_V1")) ? 1 : 0;
    // round A's sub-bucket sums for l1 jobs (one l1 candidate bucket); SIP_SEL_NOTSUM=1: counts only
    Pr.sel_tsum = (Pr.selv2 && !getenv("SIP_SEL_NOTSUM")) ? 1 : 0;
    selc_fused = Pr.selv2 && getenv("SIP_SELC_FUSED") && atoi(getenv("SIP_SELC_FUSED")) == 1;
    if (Pr.selv2) {   // k_selB / k_selC: one resident wave (the candidate regions are per CTA)
      int occ = 0;
      Pr.selb_ns = getenv("SIP_SELB_NS") ? std::min(SMAX, std::max(2, atoi(getenv("SIP_SELB_NS")))) : 2;
      CU(cudaFuncSetAttribute(k_selB<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)selb_smem(Pr.selb_ns)));
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_selB<T>, BLOCK, selb_smem(Pr.selb_ns)));
      g_sel = std::max(1, std::min(tiles, nsm * std::max(occ, 1)));
    }
    {   // pass 1 sub-ranges (tiles of BLOCK chunks; 0 = the CTA's whole range).
        // Measured: x larger than ~half of L2 (C5-L1, 268 MB) 23.6 -> 22.5 ms
        // per step with 8-tile sub-ranges; x that stays in L2 anyway (C4,
        // 33.5 MB) 2.65 -> 2.71 ms (more pipeline starts and count flushes)
      const char* e = getenv("SIP_P1_SUB");
      const bool big = (double)g.N * sizeof(T) > 64.0 * (1 << 20);
      Pr.p1_sub = (e ? atoi(e) : (big ? 8 : 0)) * BLOCK;
      const char* h = getenv("SIP_P1_HINT");
      Pr.p1_hint = h ? atoi(h) : 1;   // x (and the Alg. 2 x snapshot) evict_last: re-read by every segment
    }
    {
      const char* e1 = getenv("SIP_P1_POOL");
      const char* e2 = getenv("SIP_P1A_POOL");
      Pr.p1_pool = e1 ? std::max(2 * P1_NA_PLAIN, atoi(e1)) : 2 * P1_NA_PLAIN;
      Pr.p1a_pool = e2 ? std::max(2 * P1_NA_ADAPT, atoi(e2)) : 2 * P1_NA_ADAPT;
    }
    smem_p1v = pass1_smem(P, Pr.p1_pool, Pr.selv2);   // k_pass1t: slots + bulk-copy stage pool (+ round-A counts)
    smem_p1a = pass1_smem(P, Pr.p1a_pool, Pr.selv2);
    // pass 1: segment-major over one contiguous chunk range per CTA, one
    // resident wave (CTAs per SM from registers + stage buffers)
    {
      auto wave1 = [&](const void* fn, size_t smem, int cap) {
        int occ = 0;
        CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, BLOCK, smem));
        return std::max(1, std::min(g.N / VT<T>::W / BLOCK, nsm * std::max(1, std::min(occ, cap))));
      };
      g_p1 = wave1((const void*)k_pass1t<T, 0, 0>, smem_p1v, 3);
      g_p1a = wave1((const void*)k_pass1t<T, 1, 0>, smem_p1a, 2);
    }
    if (vec && sizeof(T) == 4) {
      // per-CTA candidate regions of the select grid: a CTA visits at most
      // ceil(chunks / (grid * BLOCK * SEL_U)) iterations of BLOCK * SEL_U chunks
      int nbmax = 1;
      for (int i = 0; i < P; ++i) if (Pr.set[i].job >= 0) nbmax = std::max(nbmax, Pr.set[i].nblk);
      const long long chunks = (long long)nbmax * (g.N / VT<T>::W);
      const long long per_it = (long long)BLOCK * SEL_U;
      const long long its = (chunks + (long long)g_sel * per_it - 1) / ((long long)g_sel * per_it);
      Pr.cand_per = its * per_it * VT<T>::W;
      // k_selB: tiles of SB_TILE chunks per operator block, strided over the grid
      const long long tiles2 = (long long)nbmax * ((g.N / VT<T>::W + SB_TILE - 1) / SB_TILE);
      const long long its2 = (tiles2 + g_sel - 1) / g_sel;
      Pr.cand_per = std::max(Pr.cand_per, its2 * SB_TILE * VT<T>::W);
      for (int i = 0; i < P; ++i) {
        const SetD<T>& S = Pr.set[i];
        if (S.job < 0) continue;
        Pr.cand[S.job] = dalloc<unsigned>((size_t)g_sel * Pr.cand_per);
        Pr.cand[S.sjob] = dalloc<unsigned>((size_t)g_sel * Pr.cand_per);
      }
    }
    Pr.ccnt = dalloc<unsigned>((size_t)MAXJOBS * std::max(g_sel, 1));
    Pr.sel_grid = g_sel;
    smem_p2 = (size_t)NWARP * P * 4 * sizeof(double);
    smem_init = (size_t)NWARP * P * 2 * sizeof(double);
    // per-fiber sets (sip_fiber.cuh): one CTA per fiber, a single wave
    if (nfib_sets) {
      int nf = 1;
      for (int i = 0; i < p; ++i) {
        const SetD<T>& S = Pr.set[i];
        if (!S.fib) continue;
        if (!S.fpath) { nfib_sort++; nf = std::max(nf, S.fib == 1 ? g.nz * g.ny : g.ny * g.nx); continue; }
        nfib_warp++;
      }
      int per = 0;
      if (nfib_sort) {
        smem_fib = fiber_smem((int)sizeof(T));
        CU(cudaFuncSetAttribute(k_fiber<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fib));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fiber<T>, BLOCK, smem_fib));
        g_fib = std::max(1, std::min(nf, nsm * std::max(per, 1)));
      }
      for (int i = 0; i < p; ++i) {   // warp kernel: one launch per set, its own single-wave grid
        const SetD<T>& S = Pr.set[i];
        if (!S.fib || !S.fpath) continue;
        auto kern = FiberW<T>::of(S.flen);
        smem_fw[i] = S.fib == 2 ? fiberw_smem(S.flen, (int)sizeof(T)) : 0;
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, BLOCK, smem_fw[i]));
        const int units = S.fib == 1 ? (g.nz * g.ny + NWARP - 1) / NWARP : g.ny * ((g.nx + FW_TC - 1) / FW_TC);
        g_fw[i] = std::max(1, std::min(units, nsm * std::max(per, 1)));
        g_fibw = std::max(g_fibw, g_fw[i]);
      }
    }
    Pr.poison = getenv("SIP_POISON") ? 1 : 0;
    Pr.init_zero = vec ? 0 : 1;
    Pr.fibv = (nfib_sets && nranks > 1) ? dalloc<double>(4 * MAXP) : nullptr;
    const int gmax = std::max({g_pts, g_sel, g_p2, g_vec, g_p1, g_cg1p, g_cg2p, g_rhsp, g_fib, g_fibw, g_svd});
    Pr.partials = dalloc<double>(std::max((size_t)(gmax + 2) * (nv1 + 8), (size_t)(g_sel + 2) * MAXJOBS * 3));
    if (nranks > 1) {   // gather slots of the z-slab finalisers (sip_team.cuh)
      int xs_ = 0;
      for (int st = ST_INIT; st <= ST_PASS2; ++st) xs_ = std::max(xs_, site_payload(st, P, njobs));
      Pr.xslot = (xs_ + 31) / 32 * 32;
      Pr.xg = dalloc<double>((size_t)nranks * Pr.xslot);
      CU(cudaMemsetAsync(Pr.xg, 0, (size_t)nranks * Pr.xslot * sizeof(double), stream));
    }
    Pr.counter = dalloc<unsigned>(1);
    CU(cudaMemsetAsync(Pr.counter, 0, sizeof(unsigned), stream));
    Pr.gf_cnt = dalloc<unsigned>((size_t)MAXJOBS * FB_N);
    Pr.gf_s0 = dalloc<unsigned long long>((size_t)MAXJOBS * FB_N);
    CU(cudaMemsetAsync(Pr.gf_cnt, 0, sizeof(unsigned) * MAXJOBS * FB_N, stream));
    CU(cudaMemsetAsync(Pr.gf_s0, 0, sizeof(unsigned long long) * MAXJOBS * FB_N, stream));
    Pr.gh_cnt = dalloc<unsigned>((size_t)MAXJOBS * NBUCK);
    Pr.gh_s0 = dalloc<unsigned long long>((size_t)MAXJOBS * NBUCK);
    Pr.gh_s1 = dalloc<unsigned long long>((size_t)MAXJOBS * NBUCK);
    Pr.gh_ta = dalloc<unsigned long long>((size_t)MAXJOBS * NBUCK);
    Pr.sel_gen = dalloc<unsigned>(1);
    CU(cudaMemsetAsync(Pr.sel_gen, 0, sizeof(unsigned), stream));
    CU(cudaMemsetAsync(Pr.gh_ta, 0, sizeof(unsigned long long) * MAXJOBS * NBUCK, stream));
    CU(cudaMemsetAsync(Pr.gh_cnt, 0, sizeof(unsigned) * MAXJOBS * NBUCK, stream));
    CU(cudaMemsetAsync(Pr.gh_s0, 0, sizeof(unsigned long long) * MAXJOBS * NBUCK, stream));
    CU(cudaMemsetAsync(Pr.gh_s1, 0, sizeof(unsigned long long) * MAXJOBS * NBUCK, stream));
    Pr.ntiles_max = 3 * tiles;
    Pr.tiecnt = dalloc<int>((size_t)std::max(njobs, 1) * Pr.ntiles_max);
    d_ctrl = dalloc<Ctrl>(1);
    Pr.ctrl = d_ctrl;
    CU(cudaMallocHost(&h_flag, 2 * sizeof(int)));
    CU(cudaEventCreateWithFlags(&ev_flag[0], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ev_flag[1], cudaEventDisableTiming));
    CU(cudaEventCreate(&ev0));
    CU(cudaEventCreate(&ev1));
    CU(cudaFuncSetAttribute(k_pass1<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CU(cudaFuncSetAttribute(k_pass1t<T, 0, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CU(cudaFuncSetAttribute(k_pass1t<T, 0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CU(cudaFuncSetAttribute(k_pass1t<T, 1, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CU(cudaFuncSetAttribute(k_pass1t<T, 1, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CU(cudaFuncSetAttribute(k_pass1t<T, 2, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    memset(&hc, 0, sizeof(hc));
    hc.njobs = njobs;
    for (int i = 0; i < P; ++i) {
      const SetD<T>& S = Pr.set[i];
      if (S.job >= 0) {
        hc.job[S.job].kind = S.kind; hc.job[S.job].set = i; hc.job[S.job].on_s = 0;
        hc.job[S.sjob].kind = S.kind; hc.job[S.sjob].set = i; hc.job[S.sjob].on_s = 1;
      }
    }
    CU(cudaStreamSynchronize(stream));
  }

  // ---- orthonormal DCT-II along every axis (reading L30) ---------------
  void setup_dct() {
    const int n[3] = {nz, ny, nx};
    bool want[2] = {false, false};
    for (int i = 0; i < p; ++i)
      if (Pr.set[i].dct) want[Pr.set[i].dct - 1] = true;
    for (int tk = 0; tk < 2; ++tk) {
      if (!want[tk]) continue;
      for (int a = 0; a < 3; ++a) {
        if (a == 1 && ndim == 2) continue;
        const int L = n[a];
        std::vector<double> h((size_t)L * L, 0.0);   // column-major D(k, j): row k = coefficient, column j = sample
        if (tk == 0) {
          for (int k = 0; k < L; ++k)
            for (int j = 0; j < L; ++j) {
              const double sc = k == 0 ? std::sqrt(1.0 / L) : std::sqrt(2.0 / L);
              h[(size_t)k + (size_t)j * L] = sc * std::cos(M_PI * (2.0 * j + 1.0) * k / (2.0 * L));
            }
        } else {
          // Haar basis, coefficient order [a_J, d_J, ..., d_1]: row 0 is the
          // constant 1/sqrt(L); the detail function at scale 2^s (support
          // 2^s samples starting at q 2^s) is +2^(-s/2) on the first half,
          // -2^(-s/2) on the second; its row is L / 2^s + q
          for (int j = 0; j < L; ++j) h[(size_t)j * L] = 1.0 / std::sqrt((double)L);
          for (int w = 2; w <= L; w *= 2) {
            const double amp = 1.0 / std::sqrt((double)w);
            for (int q = 0; q < L / w; ++q) {
              const int k = L / w + q;
              for (int t = 0; t < w; ++t) h[(size_t)k + (size_t)(q * w + t) * L] = t < w / 2 ? amp : -amp;
            }
          }
        }
        std::vector<T> ht(h.size());
        for (size_t e = 0; e < h.size(); ++e) ht[e] = (T)h[e];
        dctm[tk][a] = dalloc<T>((size_t)L * L);
        CU(cudaMemcpy(dctm[tk][a], ht.data(), ht.size() * sizeof(T), cudaMemcpyHostToDevice));
      }
    }
    dtmp = dalloc<T>((size_t)Pr.g.N);
    if (cublasCreate(&blas) != CUBLAS_STATUS_SUCCESS) throw SipError{SIP_ERR_CUDA, "cublasCreate"};
    const size_t wsb = 32u << 20;      // a fixed workspace: no allocation inside graph capture
    blas_ws = dalloc<char>(wsb);
    cublasSetWorkspace(blas, blas_ws, wsb);
    cublasSetStream(blas, stream);
    cublasSetPointerMode(blas, CUBLAS_POINTER_MODE_HOST);
  }
  T* dtmp2_ = nullptr;
  T* dtmp2() { if (!dtmp2_) dtmp2_ = dalloc<T>((size_t)Pr.g.N); return dtmp2_; }
  void gemm(cublasOperation_t ta, cublasOperation_t tb, int m_, int n_, int k_, const T* A, int lda,
            const T* B, int ldb, T* Cm, int ldc) {
    const T one = 1, zero = 0;
    cublasStatus_t st;
    if constexpr (sizeof(T) == 4)
      st = cublasSgemm(blas, ta, tb, m_, n_, k_, (const float*)&one, (const float*)A, lda, (const float*)B, ldb,
                       (const float*)&zero, (float*)Cm, ldc);
    else
      st = cublasDgemm(blas, ta, tb, m_, n_, k_, (const double*)&one, (const double*)A, lda, (const double*)B, ldb,
                       (const double*)&zero, (double*)Cm, ldc);
    if (st != CUBLAS_STATUS_SUCCESS) throw SipError{SIP_ERR_CUDA, "cuBLAS gemm failed"};
  }
  void gemm_sb(cublasOperation_t ta, cublasOperation_t tb, int m_, int n_, int k_, const T* A, int lda,
               long long sa, const T* B, int ldb, long long sb, T* Cm, int ldc, long long sc, int batch) {
    const T one = 1, zero = 0;
    cublasStatus_t st;
    if constexpr (sizeof(T) == 4)
      st = cublasSgemmStridedBatched(blas, ta, tb, m_, n_, k_, (const float*)&one, (const float*)A, lda, sa,
                                     (const float*)B, ldb, sb, (const float*)&zero, (float*)Cm, ldc, sc, batch);
    else
      st = cublasDgemmStridedBatched(blas, ta, tb, m_, n_, k_, (const double*)&one, (const double*)A, lda, sa,
                                     (const double*)B, ldb, sb, (const double*)&zero, (double*)Cm, ldc, sc, batch);
    if (st != CUBLAS_STATUS_SUCCESS) throw SipError{SIP_ERR_CUDA, "cuBLAS batched gemm failed"};
  }
  // f <- D f (inv = 0) or D^T f (inv = 1), in place through dtmp.  Column-
  // major view of the row-major field: X(x, y, z); the x axis multiplies
  // from the left, y and z from the right.
  void dct_field(T* f, int inv, int kind) {
    T* const* dm = dctm[kind - 1];
    const cublasOperation_t L_ = inv ? CUBLAS_OP_T : CUBLAS_OP_N;   // D or D^T from the left
    const cublasOperation_t R_ = inv ? CUBLAS_OP_N : CUBLAS_OP_T;   // D^T or D from the right
    gemm(L_, CUBLAS_OP_N, nx, ny * nz, nx, dm[2], nx, f, nx, dtmp, nx);                  // x
    if (ndim == 3) {
      gemm_sb(CUBLAS_OP_N, R_, nx, ny, ny, dtmp, nx, (long long)nx * ny, dm[1], ny, 0, f, nx,
              (long long)nx * ny, nz);                                                        // y, per plane
      gemm(CUBLAS_OP_N, R_, nx * ny, nz, nz, f, nx * ny, dm[0], nz, dtmp, nx * ny);        // z
    } else {
      gemm(CUBLAS_OP_N, R_, nx, nz, nz, dtmp, nx, dm[0], nz, f, nx);                       // z
      return;
    }
    CU(cudaMemcpyAsync(f, dtmp, (size_t)Pr.g.N * sizeof(T), cudaMemcpyDeviceToDevice, stream));
  }
  // the transforms around the hot-path kernels (kpos > 0: the parity of the
  // iteration, hence the y / v buffers, is known at capture time)
  void dct_after_pass1(int kpos) {
    const bool adapt = kpos % 2 == 1;
    const int par = kpos & 1;
    for (int i = 0; i < p; ++i) {
      SetD<T>& S = Pr.set[i];
      if (!S.dct) continue;
      dct_field(S.w, 0, S.dct);                             // w in the coefficient domain
      if (kpos % hc.opt.check_every == 0) dct_field(S.s, 0, S.dct);
      if (adapt) { dct_field(S.y[par ^ 1], 0, S.dct); dct_field(S.v[par ^ 1], 0, S.dct); }   // Alg. 2's k0 snapshots
    }
  }
  void dct_after_pass2(int kpos) {
    const int par = kpos & 1;
    for (int i = 0; i < p; ++i) {
      SetD<T>& S = Pr.set[i];
      if (!S.dct) continue;
      dct_field(S.y[par ^ 1], 1, S.dct);                    // y = D^T P_l1(D w), v = D^T v_c (linear)
      dct_field(S.v[par ^ 1], 1, S.dct);
    }
  }

  // per-entry bounds: compact (host, fp64) -> padded device field
  const T* upload_compact(int i, const std::vector<double>& v) {
    const SetD<T>& S = Pr.set[i];
    T* f = field(S.nblk);
    double* tmp = nullptr;
    CU(cudaMalloc(&tmp, v.size() * sizeof(double)));
    CU(cudaMemcpyAsync(tmp, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, stream));
    long long boff = 0;
    for (int b = 0; b < S.nblk; ++b) {
      k_pack<T, double><<<g_small_(), BLOCK, 0, stream>>>(Pr.g, S.prim[b], d_fmap, boff,
                                                         f + (int64_t)b * Pr.g.ld, tmp, 1);
      boff += block_len(S.prim[b]);
    }
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(stream));
    cudaFree(tmp);
    return f;
  }
  int g_small_() const { return std::max(1, std::min((Pr.g.N + BLOCK - 1) / BLOCK, nsm * 4)); }

  long long block_len(int prim) const {
    const Geo& g = Pr.g;
    switch (prim) {
      case PRIM_I: return g.N;
      case PRIM_Z: return (long long)(z0 + g.nz < nz_g ? g.nz : g.nz - 1) * g.plane;   // pad plane: last global
      case PRIM_Y: return (long long)g.nz * (g.ny - 1) * g.nx;
      case PRIM_X: return (long long)g.nz * g.ny * (g.nx - 1);
      default: {
        long long c = 0;
        for (int i = 0; i < p; ++i)
          if ((*sets)[i].op == SIP_OP_BLUR_MASK) { c = (*sets)[i].M; break; }
        return c;
      }
    }
  }
  // compact length of a block over the whole (all-slab) grid
  long long block_len_global(int prim) const {
    const Geo& g = Pr.g;
    switch (prim) {
      case PRIM_I: return (long long)nz_g * g.plane;
      case PRIM_Z: return (long long)(nz_g - 1) * g.plane;
      case PRIM_Y: return (long long)nz_g * (g.ny - 1) * g.nx;
      case PRIM_X: return (long long)nz_g * g.ny * (g.nx - 1);
      default: return block_len(prim);   // blur/mask: single rank only
    }
  }
  long long set_len_global(int i) const {
    long long c = 0;
    for (int b = 0; b < Pr.set[i].nblk; ++b) c += block_len_global(Pr.set[i].prim[b]);
    return c;
  }
  long long set_len(int i) const {
    long long c = 0;
    for (int b = 0; b < Pr.set[i].nblk; ++b) c += block_len(Pr.set[i].prim[b]);
    return c;
  }

  // ---- iteration enqueue ------------------------------------------------
  // profiling: an event is recorded before the first kernel and after every
  // kernel; consecutive pairs give each kernel's device time (kind list)
  // KB_COMM: a z-slab site's exchange + finalisers (multi-rank only)
  enum { KB_BLUR = 0, KB_RHS, KB_CG1, KB_CG2, KB_PASS1, KB_SELECT, KB_TIE, KB_PASS2, KB_CTRL, KB_COMM, KB_CGX, KB_FIBER, KB_SVD, KB_DCT, NKIND };
  bool prof = false;
  std::vector<cudaEvent_t> pev;      // events of one graph (capture order)
  std::vector<int> pkind;            // kind of the kernel ending at pev[i+1]
  size_t pev_used = 0;
  double prof_ms[NKIND] = {0};
  long long prof_cnt[NKIND] = {0};

  void mark(int kind) {
    if (!prof) return;
    if (pev_used == pev.size()) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      pev.push_back(e);
    }
    // inside stream capture the record must be an external event node
    cudaStreamCaptureStatus cs;
    CU(cudaStreamIsCapturing(stream, &cs));
    if (cs == cudaStreamCaptureStatusActive) CU(cudaEventRecordWithFlags(pev[pev_used], stream, cudaEventRecordExternal));
    else CU(cudaEventRecord(pev[pev_used], stream));
    if (pev_used > 0) pkind.push_back(kind);
    ++pev_used;
  }

  // launch with programmatic dependent launch (single rank; pdl_begin() in
  // the kernels): the next kernel is scheduled while this one drains
  bool pdl = false;
  template <typename... KA, typename... A>
  void lk(void (*kern)(KA...), int grid, int block, size_t smem, A&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = pdl ? at : nullptr;
    cfg.numAttrs = pdl ? 1 : 0;
    CU(cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...));
  }

  // kernel variants by iteration type: kpos = k (1-based) when the launch
  // position fixes it, 0 = decide on the device (see sip_pass.cuh)
  void launch_pass1(int kpos) {
    if (!vec) { k_pass1<T><<<g_pts, BLOCK, smem_p1, stream>>>(Pr); return; }
    const int ad = kpos > 0 ? (kpos % 2 == 1) : 2;
    const int ck = kpos > 0 ? (kpos % hc.opt.check_every == 0) : 2;
    switch (ad * 3 + ck) {
      case 0: lk(k_pass1t<T, 0, 0>, g_p1, BLOCK, smem_p1v, Pr); break;
      case 1: lk(k_pass1t<T, 0, 1>, g_p1, BLOCK, smem_p1v, Pr); break;
      case 3: lk(k_pass1t<T, 1, 0>, g_p1a, BLOCK, smem_p1a, Pr); break;
      case 4: lk(k_pass1t<T, 1, 1>, g_p1a, BLOCK, smem_p1a, Pr); break;
      default: lk(k_pass1t<T, 2, 2>, g_p1a, BLOCK, smem_p1a, Pr);
    }
  }
  void launch_pass2(int kpos) {
    if (!vec) { k_pass2<T><<<g_p2, BLOCK, smem_p2, stream>>>(Pr); return; }
    const int ad = kpos > 0 ? (kpos % 2 == 1) : 2;
    const int ck = kpos > 0 ? (kpos % hc.opt.check_every == 0) : 2;
    switch (ad * 3 + ck) {
      case 0: lk(k_pass2t<T, 0, 0>, g_p2, BLOCK, smem_p2, Pr); break;
      case 1: lk(k_pass2t<T, 0, 1>, g_p2, BLOCK, smem_p2, Pr); break;
      case 3: lk(k_pass2t<T, 1, 0>, g_p2, BLOCK, smem_p2, Pr); break;
      case 4: lk(k_pass2t<T, 1, 1>, g_p2, BLOCK, smem_p2, Pr); break;
      default: lk(k_pass2t<T, 2, 2>, g_p2, BLOCK, smem_p2, Pr);
    }
  }

  // ---- phase launchers (one rank's part of each step) -------------------
  void launch_blur(int mode, int j) { k_blur_t<T><<<g_pts, BLOCK, 0, stream>>>(Pr, mode, j); ++launches; }
  void launch_rhs() {
    if (vec) {
      if (ndim == 3) lk(k_rhsp<T, true>, g_rhsp, BLOCK, 0, Pr);
      else lk(k_rhsp<T, false>, g_rhsp, BLOCK, 0, Pr);
    } else k_rhs<T><<<g_pts, BLOCK, 0, stream>>>(Pr);
    ++launches;
  }
  // flat CG kernels (sip_vec.cuh k_cg1f / k_cg2f) with the deferred x update;
  // the scalar kernels (sip_kernels.cuh) for general shapes, the blur
  // operator and n_cg > MAXCG (no ring slot per step)
  bool lean_cg() const { return cgv && Pr.defer_x; }
  // small grids: one CTA runs the CG loop (at most SMALL_CG_CHUNKS 16-byte chunks)
  static constexpr int SMALL_CG_CHUNKS = 4096;
  bool small_cg() const {
    return lean_cg() && nranks == 1 && !Pr.has[PRIM_F] && Pr.g.N / VT<T>::W <= SMALL_CG_CHUNKS &&
           !getenv("SIP_NO_SMALL_CG");
  }
  const bool sel_debug = getenv("SIP_SEL_DEBUG") != nullptr;
  void launch_cg1(int j) {
    if (lean_cg()) {
      if (ndim == 3) lk(k_cg1f<T, true>, g_cg1p, BLOCK, 0, Pr, j);
      else lk(k_cg1f<T, false>, g_cg1p, BLOCK, 0, Pr, j);
    } else {
      k_cg1<T><<<g_pts, BLOCK, 0, stream>>>(Pr, j);
    }
    ++launches;
  }
  void launch_cg2(int j) {
    if (lean_cg()) {
      if (ndim == 3) lk(k_cg2f<T, true>, g_cg2p, BLOCK, 0, Pr, j);
      else lk(k_cg2f<T, false>, g_cg2p, BLOCK, 0, Pr, j);
    } else k_cg2<T><<<g_pts, BLOCK, 0, stream>>>(Pr, j);
    ++launches;
  }
  // deferred x update: one ring slot per CG step (vectorised path, n_cg <= MAXCG)
  void ensure_ring(int n_cg) {
    if (!cgv || n_cg < 1 || n_cg > MAXCG || getenv("SIP_NO_DEFER_X")) { Pr.defer_x = 0; return; }
    if (Pr.has[PRIM_F] && !Pr.ub) Pr.ub = field(1);
    while (npr < n_cg) Pr.pr[npr++] = field(1);
    Pr.defer_x = 1;
  }
  void launch_cgx() { lk(k_cgx<T>, g_vec, BLOCK, 0, Pr); ++launches; }
  void launch_select(int r) {
    if (vec) lk(k_selectf<T>, g_sel, BLOCK, 0, Pr, r);
    else k_select<T><<<g_sel, BLOCK, 0, stream>>>(Pr, r);
    ++launches;
  }
  bool has_card() const {
    for (int i = 0; i < p; ++i) if (Pr.set[i].kind == K_CARD && Pr.set[i].job >= 0) return true;
    return false;
  }
  void launch_tie() {
    if (vec) lk(k_tiecountf<T>, g_p2, BLOCK, 0, Pr);
    else k_tiecount<T><<<g_p2, BLOCK, 0, stream>>>(Pr);
    ++launches;
  }
  // per-fiber sets: one warp-kernel launch per set, the sort kernel for the rest
  void launch_fiber() {
    for (int i = 0; nfib_warp && i < p; ++i) {
      if (!Pr.set[i].fib || !Pr.set[i].fpath) continue;
      lk(FiberW<T>::of(Pr.set[i].flen), g_fw[i], BLOCK, smem_fw[i], Pr, i);
      ++launches;
    }
    if (nfib_sort) { lk(k_fiber<T>, g_fib, BLOCK, smem_fib, Pr); ++launches; }
  }
  void launch_control() { lk(k_control<T>, 1, BLOCK, 0, Pr); ++launches; }
  // rank / nuclear-norm sets: y, v of every matrix (which 0), the Eq. 26
  // numerator of s on check iterations (which 1; the kernel returns on others)
  void launch_svd_one(int i, int which, int nmat) {
    const int cl = std::max(1, svd_cl[i]);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nmat * cl));
    cfg.blockDim = dim3((unsigned)SVD_BLOCK);
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = cl > 1 ? 1 : 0;
    CU(cudaLaunchKernelEx(&cfg, k_svdproj<T>, Pr, i, which, cl));
  }
  void launch_svd() {
    for (int i = 0; i < p; ++i) {
      if (!Pr.set[i].svd) continue;
      const MatView mv = mat_view(ndim, nz_g, ny, nx, Pr.set[i].prim[0]);
      launch_svd_one(i, 0, mv.nmat); ++launches;
      launch_svd_one(i, 1, mv.nmat); ++launches;
    }
  }
  void launch_fin(int site, int j, int round) {
    k_fin<T><<<1, BLOCK, 0, stream>>>(Pr, site, j, round);
    ++launches;
  }

  void enqueue_iteration(int n_cg, int kpos = 0) {
    if (prof && pev_used == 0) mark(-1);
    if (Pr.has[PRIM_F]) { launch_blur(0, 0); mark(KB_BLUR); }
    launch_rhs(); mark(KB_RHS);
    if (small_cg()) {   // the whole CG loop in one CTA (small grids)
      if (ndim == 3) lk(k_cgsmall<T, true>, 1, BLOCK, 0, Pr, n_cg);
      else lk(k_cgsmall<T, false>, 1, BLOCK, 0, Pr, n_cg);
      ++launches; mark(KB_CG1);
    } else
    for (int j = 0; j < n_cg; ++j) {
      if (Pr.has[PRIM_F]) {
        if (lean_cg()) { lk(k_blurF<T>, g_bf, BLOCK, smem_bf, Pr, j); ++launches; }
        else launch_blur(1, j);
        mark(KB_BLUR);
      }
      launch_cg1(j); mark(KB_CG1);
      launch_cg2(j); mark(KB_CG2);
    }
    if (Pr.defer_x && n_cg > 0) { launch_cgx(); mark(KB_CGX); }
    launch_pass1(kpos);
    ++launches; mark(KB_PASS1);
    if (ndct_sets) {
      if (kpos <= 0) throw SipError{SIP_ERR_CONFIG, "transform-domain sets need graph_iters a multiple of lcm(2, check_every) (or 0)"};
      dct_after_pass1(kpos); mark(KB_DCT);
    }
    if (hc.njobs > 0) {
      if (sel_small) {
        lk(k_selsmall<T>, hc.njobs, BLOCK, selsmall_smem(), Pr); ++launches; mark(KB_SELECT);
      } else if (Pr.selv2) {   // one streaming pass + candidate rounds (round A ran in pass 1)
        lk(k_selB<T>, g_sel, BLOCK, selb_smem(Pr.selb_ns), Pr); ++launches; mark(KB_SELECT);
        if (selc_fused) { lk(k_selCF<T>, g_sel, BLOCK, 0, Pr); ++launches; mark(KB_SELECT); }
        else for (int r = 2; r <= 4; ++r) { lk(k_selC<T>, g_sel, BLOCK, 0, Pr, r); ++launches; mark(KB_SELECT); }
      } else {
        for (int r = 1; r <= KeyT<T>::ROUNDS; ++r) { launch_select(r); mark(KB_SELECT); }
      }
      if (sel_debug) k_seldbg<T><<<1, 32, 0, stream>>>(Pr);
      if (has_card()) { launch_tie(); mark(KB_TIE); }
    }
    if (Pr.nseg2 > 0) {
      launch_pass2(kpos);
      ++launches; mark(KB_PASS2);
    }
    if (ndct_sets) { dct_after_pass2(kpos); mark(KB_DCT); }
    if (nfib_sets) { launch_fiber(); mark(KB_FIBER); }   // per-fiber projections, after pass 2's sums
    if (nsvd_sets) { launch_svd(); mark(KB_SVD); }       // rank / nuclear-norm sets
    launch_control(); mark(KB_CTRL);
  }

  void harvest_profile() {
    if (!prof || pev_used < 2) return;
    CU(cudaEventSynchronize(pev[pev_used - 1]));
    for (size_t i = 0; i + 1 < pev_used; ++i) {
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, pev[i], pev[i + 1]));
      prof_ms[pkind[i]] += ms;
      prof_cnt[pkind[i]] += 1;
    }
  }

  void ensure_graph(int iters, int n_cg) {
    if (gexec && g_iters == iters && g_ncg == n_cg && g_prof == prof && g_ce == hc.opt.check_every) return;
    if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
    cudaGraph_t graph;
    long long before = launches;
    pev_used = 0;
    pkind.clear();
    apply_l2_window();   // captured into the kernel nodes
    CU(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    // the adapt / check pattern repeats every lcm(2, check_every) iterations
    const int ce = std::max(1, hc.opt.check_every);
    const int period = (ce % 2 == 0) ? ce : 2 * ce;
    const bool fixed = (iters % period == 0);
    for (int i = 0; i < iters; ++i) enqueue_iteration(n_cg, fixed ? i + 1 : 0);
    cudaError_t e = cudaStreamEndCapture(stream, &graph);
    if (e != cudaSuccess) throw SipError{SIP_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e)};
    graph_kernels = launches - before;
    launches = before;
    CU(cudaGraphInstantiate(&gexec, graph, 0));
    cudaGraphDestroy(graph);
    g_iters = iters;
    g_ncg = n_cg;
    g_prof = prof;
    g_ce = hc.opt.check_every;
  }

  void ensure_log(int max_iter) {
    if (log_cap >= max_iter) return;
    log_cap = max_iter;
    d_log_cg = dalloc<int>(max_iter);
    d_log_br = dalloc<int>((size_t)max_iter * P);
    d_log_rho = dalloc<double>((size_t)max_iter * P);
    d_log_gam = dalloc<double>((size_t)max_iter * P);
    d_log_feas = dalloc<double>((size_t)max_iter * std::max(p, 1));
    d_log_evol = dalloc<double>(max_iter);
    d_log_supp = dalloc<unsigned long long>((size_t)max_iter * std::max(p, 1));
  }

  // ---- control block -----------------------------------------------------
  void fill_ctrl(const Options& o, int max_iter, double eps_feas, double eps_evol, double floor_,
                 const double* rho_in, const double* gamma_in) {
    Ctrl c = hc;   // keeps job kinds/sets
    c.k = 1; c.stopped = 0; c.converged = 0; c.first_adapt_done = 0; c.adapt_calls = 0;
    c.hist_head = 0; c.hist_count = 1; c.breakdown = 0; c.numeric_err = 0; c.zero_x = 0;
    c.cg_j = 0; c.cg_active = 0; c.cg_count = 0; c.cg_total = 0;
    c.P = P; c.p = p;
    c.opt.n_cg = o.n_cg; c.opt.eq25 = o.eq25; c.opt.fixed_work = o.fixed_work;
    c.opt.adapt_every = o.adapt_every; c.opt.check_every = o.check_every; c.opt.max_iter = max_iter;
    c.opt.eps_evol = eps_evol; c.opt.eps_feas = eps_feas; c.opt.eps_corr = o.eps_corr;
    c.opt.rho_ratio_cap = o.rho_ratio_cap; c.opt.gamma_max = o.gamma_max; c.opt.cg_tol_floor = floor_;
    for (int i = 0; i < P; ++i) {
      c.rho[i] = rho_in ? rho_in[i] : o.rho0;
      c.gamma[i] = gamma_in ? gamma_in[i] : o.gamma0;
    }
    for (int i = 0; i < p; ++i) {
      const HostSet& hs = (*sets)[i];
      c.u_sigma[i] = hs.prm.sigma;
      c.u_sig_lo[i] = hs.prm.sigma_lo;
      c.u_sig_hi[i] = hs.prm.sigma_hi;
      c.u_kfrac[i] = hs.prm.k_frac;
      c.u_k[i] = hs.prm.k;
      c.rel[i] = hs.prm.relative;
      c.zin[i] = hs.zero_in;
      c.mreal[i] = Pr.set[i].fib ? Pr.set[i].flen : set_len_global(i);   // per fiber for fiber sets
    }
    c.mreal[p] = (long long)nz_g * Pr.g.plane;
    make_coeffs(Pr, c.rho, &c.cI, &c.cz, &c.cy, &c.cx, &c.cF);
    c.log_cg = d_log_cg; c.log_branch = d_log_br; c.log_rho = d_log_rho; c.log_gamma = d_log_gam;
    c.log_feas = d_log_feas; c.log_evol = d_log_evol; c.log_supp = d_log_supp; c.log_len = log_cap;
    hc = c;
    CU(cudaMemcpyAsync(d_ctrl, &hc, sizeof(Ctrl), cudaMemcpyHostToDevice, stream));
  }

  void fill_logs_nan(int max_iter) {
    k_fill<int><<<g_small_(), BLOCK, 0, stream>>>(d_log_br, (long long)max_iter * P, -1);
    k_fill<double><<<g_small_(), BLOCK, 0, stream>>>(d_log_feas, (long long)max_iter * std::max(p, 1), NAN);
    k_fill<double><<<g_small_(), BLOCK, 0, stream>>>(d_log_evol, (long long)max_iter, NAN);
    k_fill<int><<<g_small_(), BLOCK, 0, stream>>>(d_log_cg, (long long)max_iter, 0);
    CU(cudaMemsetAsync(d_log_supp, 0, (size_t)max_iter * std::max(p, 1) * sizeof(unsigned long long), stream));
  }

  // init_yv: 1 = y_i = A_i m, v_i = 0; 0 = keep Y[1]/V[1] (prolonged / warm)
  void run_init(int init_x, int init_yv) {
    if (vec && !getenv("SIP_SCALAR_INIT")) k_initv<T><<<g_vec, BLOCK, smem_init, stream>>>(Pr, init_x, init_yv);
    else k_init<T><<<g_pts, BLOCK, smem_init, stream>>>(Pr, init_x, init_yv);
    ++launches;
  }

  // replay graphs until the device says stopped (lagged poll)
  void run_iterations(int max_iter, int gi, int n_cg) {
    if (gi <= 0) {
      // no graph: launch iteration by iteration, poll every check_every
      for (int it = 0; it < max_iter; ++it) {
        if (prof) { pev_used = 0; pkind.clear(); }
        enqueue_iteration(n_cg, it + 1);
        harvest_profile();
        if ((it + 1) % std::max(1, hc.opt.check_every) == 0 || it + 1 == max_iter) {
          CU(cudaMemcpyAsync(h_flag, &d_ctrl->stopped, sizeof(int), cudaMemcpyDeviceToHost, stream));
          CU(cudaStreamSynchronize(stream));
          if (h_flag[0]) break;
        }
      }
      return;
    }
    ensure_graph(gi, n_cg);
    const int nlaunch = (max_iter + gi - 1) / gi;
    const bool poll = !hc.opt.fixed_work;
    for (int l = 0; l < nlaunch; ++l) {
      CU(cudaGraphLaunch(gexec, stream));
      launches += graph_kernels;
      harvest_profile();
      if (!poll) continue;
      CU(cudaMemcpyAsync(&h_flag[l & 1], &d_ctrl->stopped, sizeof(int), cudaMemcpyDeviceToHost, stream));
      CU(cudaEventRecord(ev_flag[l & 1], stream));
      if (l >= 1) {
        CU(cudaEventSynchronize(ev_flag[(l - 1) & 1]));
        if (h_flag[(l - 1) & 1]) break;
      }
    }
  }

  void read_ctrl() {
    CU(cudaMemcpyAsync(&hc, d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, stream));
    CU(cudaStreamSynchronize(stream));
  }

  // full single-level solve on the engine's m; x result stays in Pr.x
  void solve(const Options& o, int max_iter, double eps_feas, double eps_evol, int init_x, int init_yv,
             const double* rho_in, const double* gamma_in) {
    ensure_log(max_iter);
    ensure_ring(o.n_cg);
    const double floor_ = o.cg_tol_floor > 0 ? o.cg_tol_floor
                                             : 10.0 * (sizeof(T) == 4 ? (double)FLT_EPSILON : DBL_EPSILON);
    fill_ctrl(o, max_iter, eps_feas, eps_evol, floor_, rho_in, gamma_in);
    fill_logs_nan(max_iter);
    run_init(init_x, init_yv);
    for (int i = 0; i < p; ++i) {   // relative transform-domain radius: sigma = frac ||D m||_1 (reading L30)
      if (!(Pr.set[i].dct && (*sets)[i].prm.relative)) continue;
      CU(cudaMemcpyAsync(dtmp2(), Pr.m, (size_t)Pr.g.N * sizeof(T), cudaMemcpyDeviceToDevice, stream));
      dct_field(dtmp2(), 0, Pr.set[i].dct);
      k_dct_sigma<T><<<g_small_(), BLOCK, 0, stream>>>(Pr, i, dtmp2());
      ++launches;
    }
    for (int i = 0; i < p; ++i) {   // relative nuclear-norm radius: sigma = frac ||A m||_* (y = A m after init)
      if (!(Pr.set[i].kind == K_NUC && (*sets)[i].prm.relative)) continue;
      if (!init_yv) throw SipError{SIP_ERR_CONFIG, "relative nuclear-norm radius needs y = A m at the start (no warm start / multilevel)"};
      const MatView mv = mat_view(ndim, nz_g, ny, nx, Pr.set[i].prim[0]);
      launch_svd_one(i, 2, mv.nmat);
      ++launches;
    }
    run_iterations(max_iter, o.graph_iters, o.n_cg);
    read_ctrl();
    check_canaries();
    ran = true;
    scratch_used = false;
  }

  void fill_result(sip_result* r, float ms) {
    if (!r) return;
    memset(r, 0, sizeof(*r));
    r->iterations = std::min(hc.k, hc.opt.max_iter);
    r->cg_iterations = hc.cg_total;
    r->converged = hc.converged;
    r->breakdown = hc.breakdown;
    r->r_evol = hc.r_evol;
    r->ms = ms;
    for (int i = 0; i < p; ++i) r->r_feas[i] = hc.r_feas[i];
    for (int i = 0; i < P; ++i) { r->rho[i] = hc.rho[i]; r->gamma[i] = hc.gamma[i]; }
  }

  // device field block (of the final parity) of set i
  T* final_field(int i, int which) {
    // the last iteration k wrote parity (k+1)&1; if stopped by max_iter the
    // control kernel advanced k past max_iter (k = max_iter + 1)
    const int kk = std::min(hc.k, hc.opt.max_iter);
    const int par = (kk + 1) & 1;
    return which == 0 ? Pr.set[i].y[par] : Pr.set[i].v[par];
  }

  // make the final y/v the k = 1 read buffers (warm start / multilevel source)
  void rotate_final_to_read() {
    const int kk = std::min(hc.k, hc.opt.max_iter);
    const int par = (kk + 1) & 1;
    if (par == 1) return;
    for (int i = 0; i < P; ++i) {
      SetD<T>& S = Pr.set[i];
      std::swap(S.y[0], S.y[1]);
      std::swap(S.v[0], S.v[1]);
    }
    if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }   // params changed
  }
};

// ------------------------------------------------------------------ z slabs
// Slab rule: nz planes split as evenly as possible, the first
// nz mod G ranks holding one extra plane.
inline void slab_of(int nz, int G, int r, int* z0, int* n) {
  const int q = nz / G, m = nz % G;
  *n = q + (r < m ? 1 : 0);
  *z0 = r * q + std::min(r, m);
}

// NCCL, resolved at run time (the library loads without it; a multi-rank grid
// needs it).  Only the stable C API is used: unique id, init, send/recv in
// groups, destroy.  With torch imported first, its libnccl.so.2 is reused.
typedef struct { char internal[128]; } nccl_uid;
typedef void* nccl_comm_t;
enum { NCCL_CHAR = 0 };
struct NcclApi {
  bool ok = false;
  std::string err;
  int (*GetUniqueId)(nccl_uid*) = nullptr;
  int (*CommInitRank)(nccl_comm_t*, int, nccl_uid, int) = nullptr;
  int (*CommDestroy)(nccl_comm_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
NcclApi& nccl() {
  static NcclApi a = [] {
    NcclApi n;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) { n.err = std::string("libnccl.so.2 not found: ") + dlerror(); return n; }
    auto sym = [&](const char* s) { return dlsym(h, s); };
    n.GetUniqueId = (int (*)(nccl_uid*))sym("ncclGetUniqueId");
    n.CommInitRank = (int (*)(nccl_comm_t*, int, nccl_uid, int))sym("ncclCommInitRank");
    n.CommDestroy = (int (*)(nccl_comm_t))sym("ncclCommDestroy");
    n.Send = (int (*)(const void*, size_t, int, int, nccl_comm_t, cudaStream_t))sym("ncclSend");
    n.Recv = (int (*)(void*, size_t, int, int, nccl_comm_t, cudaStream_t))sym("ncclRecv");
    n.GroupStart = (int (*)())sym("ncclGroupStart");
    n.GroupEnd = (int (*)())sym("ncclGroupEnd");
    n.GetErrorString = (const char* (*)(int))sym("ncclGetErrorString");
    n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.Send && n.Recv && n.GroupStart &&
           n.GroupEnd && n.GetErrorString;
    if (!n.ok) n.err = "libnccl.so.2 lacks the send/recv API";
    return n;
  }();
  return a;
}
#define NC(call)                                                                              \
  do {                                                                                        \
    int r_ = (call);                                                                          \
    if (r_ != 0) throw SipError{SIP_ERR_NCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)}; \
  } while (0)

// one plane transfer of a field block (element pointers as bytes)
enum { H_LO = 1,    // fill my lower ghost plane (z0 - 1) from the rank below
       H_HI = 2,    // fill my upper ghost plane (z0 + nz) from the rank above
       H_BOTH = 3 };
struct PlaneX {
  char *lo_ghost, *first, *last, *hi_ghost;
  size_t bytes;
  int dir;
};

// The exchange step of a site: halos of the listed planes plus the gather of
// every rank's slot (n doubles at slot r of rank r's buffer) to all ranks.
// xf[l] / xg[l]: the planes and gather buffer of the l-th LOCAL rank.
struct Comm {
  int G = 1;
  virtual ~Comm() {}
  virtual void exchange(const std::vector<std::vector<PlaneX>>& xf, const std::vector<double*>& xg,
                        size_t slot, size_t n, cudaStream_t st) = 0;
};

// All G slabs on this device (option "virtual_ranks"): the same decomposition,
// finalisers and exchange schedule as the NCCL path, the transfers as device
// copies on the grid's stream (captured into the iteration graph).
struct LocalComm : Comm {
  void exchange(const std::vector<std::vector<PlaneX>>& xf, const std::vector<double*>& xg, size_t slot,
                size_t n, cudaStream_t st) override {
    for (int r = 0; r < G; ++r)
      for (size_t k = 0; k < xf[r].size(); ++k) {
        const PlaneX& X = xf[r][k];
        if ((X.dir & H_LO) && r > 0)
          CU(cudaMemcpyAsync(X.lo_ghost, xf[r - 1][k].last, X.bytes, cudaMemcpyDeviceToDevice, st));
        if ((X.dir & H_HI) && r < G - 1)
          CU(cudaMemcpyAsync(X.hi_ghost, xf[r + 1][k].first, X.bytes, cudaMemcpyDeviceToDevice, st));
      }
    if (n)
      for (int r = 0; r < G; ++r)
        for (int q = 0; q < G; ++q)
          if (q != r)
            CU(cudaMemcpyAsync(xg[q] + r * slot, xg[r] + r * slot, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
};

// One rank per GPU: one NCCL group per site (grouped send/recv: the halo
// planes with the z neighbours, the slot with every peer).  Sends and
// receives between a pair are issued in the same order on both sides.
struct NcclComm : Comm {
  int rank = 0;
  nccl_comm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  void exchange(const std::vector<std::vector<PlaneX>>& xf, const std::vector<double*>& xg, size_t slot,
                size_t n, cudaStream_t st) override {
    if (xf[0].empty() && !n) return;
    NcclApi& A = nccl();
    NC(A.GroupStart());
    for (const PlaneX& X : xf[0]) {
      if (X.dir & H_LO) {
        if (rank > 0) NC(A.Recv(X.lo_ghost, X.bytes, NCCL_CHAR, rank - 1, comm, st));
        if (rank < G - 1) NC(A.Send(X.last, X.bytes, NCCL_CHAR, rank + 1, comm, st));
      }
      if (X.dir & H_HI) {
        if (rank < G - 1) NC(A.Recv(X.hi_ghost, X.bytes, NCCL_CHAR, rank + 1, comm, st));
        if (rank > 0) NC(A.Send(X.first, X.bytes, NCCL_CHAR, rank - 1, comm, st));
      }
    }
    if (n)
      for (int q = 0; q < G; ++q) {
        if (q == rank) continue;
        NC(A.Send(xg[0] + rank * slot, n * sizeof(double), NCCL_CHAR, q, comm, st));
        NC(A.Recv(xg[0] + q * slot, n * sizeof(double), NCCL_CHAR, q, comm, st));
      }
    NC(A.GroupEnd());
  }
};

// fields whose planes a site exchanges
enum FieldSel { FS_X, FS_R, FS_M, FS_Y0, FS_Y1, FS_V0, FS_V1, FS_PRING /* + slot: p ring (pr) */ };
enum SetSel { SS_ALL = 0, SS_POINTWISE = 1, SS_GLOBAL = 2, SS_ALLBLK = 3 /* every block of every set */ };
struct HaloReq { int sel, sets, dir; };

// The engines of this process's ranks (1 with NCCL, G with virtual ranks) run
// each step in lock-step: every engine launches its part, then the site's
// exchange, then every engine's k_fin.  The whole iteration is one CUDA graph.
template <class T>
struct Team : EngineBase {
  std::vector<std::unique_ptr<Engine<T>>> eng;
  Comm* comm = nullptr;
  int G = 1;
  cudaStream_t stream = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int g_iters = 0, g_ncg = -1, g_ce = 0;
  bool g_prof = false;
  long long launches = 0, graph_kernels = 0;
  int* h_flag = nullptr;
  cudaEvent_t ev_flag[2];
  bool ran = false;

  ~Team() override {
    if (gexec) cudaGraphExecDestroy(gexec);
    if (h_flag) cudaFreeHost(h_flag);
    cudaEventDestroy(ev_flag[0]); cudaEventDestroy(ev_flag[1]);
  }

  // ranks [r0, r0 + nlocal) of G live in this process
  void setup(int ndim, int nz_g, int ny, int nx, const double* h, cudaStream_t st, const std::vector<HostSet>& s,
             int G_, int r0, int nlocal, Comm* c) {
    G = G_; comm = c; stream = st;
    for (const HostSet& hs : s)   // x-fibers lie in a plane, z-fibers cross the slabs
      if (hs.fib == SIP_APPLY_Z_FIBERS) throw SipError{SIP_ERR_CONFIG, "z-fiber sets on z slabs: not in this build"};
    for (const HostSet& hs : s)
      if (!hs.lo_vec.empty() || !hs.hi_vec.empty())
        throw SipError{SIP_ERR_CONFIG, "per-entry bounds on z slabs: not in this build"};
    for (int l = 0; l < nlocal; ++l) {
      int z0, nzl;
      slab_of(nz_g, G, r0 + l, &z0, &nzl);
      if (nzl < 1) throw SipError{SIP_ERR_CONFIG, "fewer z planes than ranks"};
      auto e = std::make_unique<Engine<T>>();
      e->setup(ndim, nzl, ny, nx, h, st, s, z0, nz_g, G, r0 + l);
      if (!e->vec)
        throw SipError{SIP_ERR_CONFIG, "multi-rank grids need nx % (16 / sizeof(dtype)) == 0 and no blur/mask operator"};
      eng.push_back(std::move(e));
    }
    CU(cudaMallocHost(&h_flag, 2 * sizeof(int)));
    CU(cudaEventCreateWithFlags(&ev_flag[0], cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&ev_flag[1], cudaEventDisableTiming));
  }

  void add_planes(Engine<T>& e, const HaloReq& q, std::vector<PlaneX>& out) {
    const Geo& g = e.Pr.g;
    const size_t pl = (size_t)g.plane;
    auto push = [&](T* b) {
      PlaneX X;
      X.lo_ghost = (char*)(b - pl);
      X.first = (char*)b;
      X.last = (char*)(b + (size_t)(g.nz - 1) * pl);
      X.hi_ghost = (char*)(b + (size_t)g.nz * pl);
      X.bytes = pl * sizeof(T);
      X.dir = q.dir;
      out.push_back(X);
    };
    switch (q.sel) {
      case FS_X: push(e.Pr.x); return;
      case FS_R: push(e.Pr.r); return;
      case FS_M: push(const_cast<T*>(e.Pr.m)); return;
      default: break;
    }
    if (q.sel >= FS_PRING) { push(e.Pr.pr[q.sel - FS_PRING]); return; }
    const bool isy = q.sel == FS_Y0 || q.sel == FS_Y1;
    const int par = (q.sel == FS_Y1 || q.sel == FS_V1) ? 1 : 0;
    for (int i = 0; i < e.P; ++i) {
      SetD<T>& S = e.Pr.set[i];
      if (q.sets == SS_POINTWISE && S.global) continue;
      if (q.sets == SS_GLOBAL && !S.global) continue;
      for (int b = 0; b < S.nblk; ++b)   // only D_z blocks reach across planes (D_z^T in the rhs)
        if (S.prim[b] == PRIM_Z || q.sets == SS_ALLBLK) push((isy ? S.y[par] : S.v[par]) + (int64_t)b * g.ld);
    }
  }

  // exchange (halos + gather of `site`'s payload) and the finalisers
  void site(int st_, int j, int round, std::initializer_list<HaloReq> reqs, bool fin = true) {
    std::vector<std::vector<PlaneX>> xf(eng.size());
    std::vector<double*> xg(eng.size());
    for (size_t l = 0; l < eng.size(); ++l) {
      for (const HaloReq& q : reqs) add_planes(*eng[l], q, xf[l]);
      xg[l] = eng[l]->Pr.xg;
    }
    const size_t n = fin ? (size_t)site_payload(st_, eng[0]->P, eng[0]->hc.njobs) : 0;
    comm->exchange(xf, xg, (size_t)eng[0]->Pr.xslot, n, stream);
    if (fin)
      for (auto& e : eng) { e->launch_fin(st_, j, round); ++launches; }
    eng[0]->mark(Engine<T>::KB_COMM);
  }

  template <class F>
  void each(F&& f, int kind = -1) {
    for (auto& e : eng) { long long b = e->launches; f(*e); launches += e->launches - b; }
    if (kind >= 0) eng[0]->mark(kind);
  }

  // one outer iteration; kpos (1-based position in the 10-iteration pattern)
  // fixes the y / v parity and the iteration type at capture
  void enqueue_iteration(int n_cg, int kpos) {
    const int wr = (kpos & 1) ^ 1;   // parity written by this iteration
    Engine<T>& e0 = *eng[0];
    if (e0.prof && e0.pev_used == 0) e0.mark(-1);
    using E = Engine<T>;
    each([&](Engine<T>& e) { e.launch_rhs(); }, E::KB_RHS);
    site(ST_RHS, 0, 0, {{FS_R, 0, H_BOTH}});
    for (int j = 0; j < n_cg; ++j) {
      each([&](Engine<T>& e) { e.launch_cg1(j); }, E::KB_CG1);
      site(ST_CG1, j, 0, {{FS_PRING + (e0.Pr.defer_x ? j : (j & 1)), 0, H_BOTH}});
      each([&](Engine<T>& e) { e.launch_cg2(j); }, E::KB_CG2);
      if (j == n_cg - 1 && !e0.Pr.defer_x) site(ST_CG2, j, 0, {{FS_X, 0, H_BOTH}});   // x^{k+1} for pass 1, next rhs
      else site(ST_CG2, j, 0, {{FS_R, 0, H_BOTH}});
    }
    if (e0.Pr.defer_x && n_cg > 0) {
      each([&](Engine<T>& e) { e.launch_cgx(); }, E::KB_CGX);
      site(ST_CG2, 0, 0, {{FS_X, 0, H_BOTH}}, false);
    }
    each([&](Engine<T>& e) { e.launch_pass1(kpos); ++e.launches; }, E::KB_PASS1);
    site(ST_PASS1, 0, 0, {{wr ? FS_Y1 : FS_Y0, SS_POINTWISE, H_LO}, {wr ? FS_V1 : FS_V0, SS_POINTWISE, H_LO}});
    if (e0.hc.njobs > 0) {
      for (int r = 1; r <= KeyT<T>::ROUNDS; ++r) {
        each([&](Engine<T>& e) { e.launch_select(r); }, E::KB_SELECT);
        site(ST_SELECT, 0, r, {});
      }
      if (e0.has_card()) {
        each([&](Engine<T>& e) { e.launch_tie(); }, E::KB_TIE);
        site(ST_TIE, 0, 0, {});
      }
    }
    if (e0.nfib_sets)   // before pass 2: its finaliser adds the fiber sums (Prob::fibv)
      each([&](Engine<T>& e) { e.launch_fiber(); }, E::KB_FIBER);
    if (e0.Pr.nglob > 0) {
      each([&](Engine<T>& e) { e.launch_pass2(kpos); ++e.launches; }, E::KB_PASS2);
      site(ST_PASS2, 0, 0, {{wr ? FS_Y1 : FS_Y0, SS_GLOBAL, H_LO}, {wr ? FS_V1 : FS_V0, SS_GLOBAL, H_LO}});
    }
    each([&](Engine<T>& e) { e.launch_control(); }, E::KB_CTRL);
  }

  int period() const {
    const int ce = std::max(1, eng[0]->hc.opt.check_every);
    return (ce % 2 == 0) ? ce : 2 * ce;
  }

  void ensure_graph(int iters, int n_cg) {
    const int ce = eng[0]->hc.opt.check_every;
    if (gexec && g_iters == iters && g_ncg == n_cg && g_ce == ce && g_prof == eng[0]->prof) return;
    if (gexec) { cudaGraphExecDestroy(gexec); gexec = nullptr; }
    cudaGraph_t graph;
    const long long before = launches;
    eng[0]->pev_used = 0;
    eng[0]->pkind.clear();
    eng[0]->apply_l2_window();
    CU(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < iters; ++i) enqueue_iteration(n_cg, i + 1);
    cudaError_t e = cudaStreamEndCapture(stream, &graph);
    if (e != cudaSuccess) throw SipError{SIP_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e)};
    graph_kernels = launches - before;
    launches = before;
    CU(cudaGraphInstantiate(&gexec, graph, 0));
    cudaGraphDestroy(graph);
    g_iters = iters; g_ncg = n_cg; g_ce = ce; g_prof = eng[0]->prof;
  }

  void run_iterations(int max_iter, int gi, int n_cg) {
    const bool poll = !eng[0]->hc.opt.fixed_work;
    int* d_stop = &eng[0]->d_ctrl->stopped;
    if (gi <= 0) {
      for (int it = 0; it < max_iter; ++it) {
        if (eng[0]->prof) { eng[0]->pev_used = 0; eng[0]->pkind.clear(); }
        enqueue_iteration(n_cg, it + 1);
        eng[0]->harvest_profile();
        if ((it + 1) % std::max(1, eng[0]->hc.opt.check_every) == 0 || it + 1 == max_iter) {
          CU(cudaMemcpyAsync(h_flag, d_stop, sizeof(int), cudaMemcpyDeviceToHost, stream));
          CU(cudaStreamSynchronize(stream));
          if (h_flag[0]) break;
        }
      }
      return;
    }
    const int per = period();
    gi = (gi + per - 1) / per * per;   // the graph must start every launch at the same pattern position
    ensure_graph(gi, n_cg);
    const int nlaunch = (max_iter + gi - 1) / gi;
    for (int l = 0; l < nlaunch; ++l) {
      CU(cudaGraphLaunch(gexec, stream));
      launches += graph_kernels;
      eng[0]->harvest_profile();
      if (!poll) continue;
      CU(cudaMemcpyAsync(&h_flag[l & 1], d_stop, sizeof(int), cudaMemcpyDeviceToHost, stream));
      CU(cudaEventRecord(ev_flag[l & 1], stream));
      if (l >= 1) {
        CU(cudaEventSynchronize(ev_flag[(l - 1) & 1]));
        if (h_flag[(l - 1) & 1]) break;
      }
    }
  }

  // single-level solve on the engines' m slabs (Algorithm 1)
  void solve(const Options& o, int max_iter, double eps_feas, double eps_evol, int init_x, int init_yv,
             const double* rho_in, const double* gamma_in) {
    const double floor_ = o.cg_tol_floor > 0 ? o.cg_tol_floor
                                             : 10.0 * (sizeof(T) == 4 ? (double)FLT_EPSILON : DBL_EPSILON);
    launches = 0;
    each([&](Engine<T>& e) {
      e.ensure_log(max_iter);
      e.ensure_ring(o.n_cg);
      e.fill_ctrl(o, max_iter, eps_feas, eps_evol, floor_, rho_in, gamma_in);
      e.fill_logs_nan(max_iter);
    });
    // halos of m (A m in k_init) and of a given x
    if (init_x) site(ST_INIT, 0, 0, {{FS_M, 0, H_BOTH}}, false);
    else site(ST_INIT, 0, 0, {{FS_M, 0, H_BOTH}, {FS_X, 0, H_BOTH}}, false);
    each([&](Engine<T>& e) { e.run_init(init_x, init_yv); });
    site(ST_INIT, 0, 0, {{FS_X, 0, H_BOTH}, {FS_Y1, SS_ALL, H_LO}, {FS_V1, SS_ALL, H_LO}});
    run_iterations(max_iter, o.graph_iters, o.n_cg);
    each([&](Engine<T>& e) { e.read_ctrl(); e.check_canaries(); e.ran = true; e.scratch_used = false; });
    ran = true;
  }
};

}  // namespace

// ------------------------------------------------------------------ grid
struct sip_grid_s {
  int device = 0;
  cudaStream_t stream = nullptr;        // library-owned work stream (capturable)
  cudaStream_t user_stream = nullptr;   // caller's stream: work is ordered after it
  cudaEvent_t fence = nullptr;
  sip_dtype dtype = SIP_F32;
  int ndim = 2;
  int64_t n[3] = {1, 1, 1};   // nz, ny, nx
  double h[3] = {1, 1, 1};
  int nranks = 1, rank = 0;   // NCCL z-slab decomposition (one rank per process)
  int vranks = 1;             // option "virtual_ranks": G slabs on this device
  std::unique_ptr<Comm> comm;
  std::vector<HostSet> sets;
  Options opt;
  std::string err;
  std::unique_ptr<EngineBase> eng;                 // single-level engine
  EngineBase* last = nullptr;                      // engine of the last projection (finest level)
  EngineBase* last_team = nullptr;                 // z slabs: Team of the last projection (finest level)
  std::vector<std::unique_ptr<EngineBase>> levels; // multilevel (index 0 = finest)
  std::unique_ptr<EngineBase> dyk;                 // sip_dykstra's sub-engines (kept alive until the next call)
  bool have_m = false;
  long long last_launches = 0;
};

namespace {

template <class T>
Engine<T>* engine_of(sip_grid g) {
  if (g->nranks > 1 || g->vranks > 1)
    throw SipError{SIP_ERR_CONFIG, "step-level entry points and multilevel are single-rank in this build"};
  if (!g->eng) {
    auto e = std::make_unique<Engine<T>>();
    e->setup(g->ndim, (int)g->n[0], (int)g->n[1], (int)g->n[2], g->h, g->stream, g->sets);
    g->eng = std::move(e);
  }
  return static_cast<Engine<T>*>(g->eng.get());
}

template <class T>
void copy_in(Engine<T>* e, const void* src, T* dst, size_t n) {
  CU(cudaMemcpyAsync(dst, src, n * sizeof(T), is_device_ptr(src) ? cudaMemcpyDeviceToDevice
                                                                  : cudaMemcpyHostToDevice, e->stream));
}
template <class T>
void copy_out(Engine<T>* e, const T* src, void* dst, size_t n) {
  CU(cudaMemcpyAsync(dst, src, n * sizeof(T), is_device_ptr(dst) ? cudaMemcpyDeviceToDevice
                                                                  : cudaMemcpyDeviceToHost, e->stream));
}

double eps_evol_of(const sip_grid g, double tol) {
  if (g->opt.eps_evol > 0) return g->opt.eps_evol;
  return tol > 0 ? 10.0 * tol : 1e-2;
}

bool is_team(const sip_grid g) { return g->nranks > 1 || g->vranks > 1; }

template <class T>
Team<T>* team_of(sip_grid g) {
  if (!g->eng) {
    const bool nc = g->nranks > 1;
    const int G = nc ? g->nranks : g->vranks;
    if (!nc && !g->comm) {
      auto lc = std::make_unique<LocalComm>();
      lc->G = G;
      g->comm = std::move(lc);
    }
    auto t = std::make_unique<Team<T>>();
    t->setup(g->ndim, (int)g->n[0], (int)g->n[1], (int)g->n[2], g->h, g->stream, g->sets, G,
             nc ? g->rank : 0, nc ? 1 : G, g->comm.get());
    g->eng = std::move(t);
  }
  return static_cast<Team<T>*>(g->eng.get());
}

// z-slab projection: NCCL ranks (m, x = this rank's slab) or virtual ranks
// (m, x = the whole grid, slab l at plane offset z0_l)
template <class T>
sip_status project_team_T(sip_grid g, const void* m, void* x, int max_iter, double tol, sip_result* res) {
  Team<T>* t = team_of<T>(g);
  Engine<T>* e0 = t->eng[0].get();
  const double eps_feas = tol > 0 ? tol : 1e-3;
  e0->prof = g->opt.profile != 0;
  for (int q = 0; q < Engine<T>::NKIND; ++q) { e0->prof_ms[q] = 0; e0->prof_cnt[q] = 0; }
  CU(cudaEventRecord(e0->ev0, g->stream));
  const int64_t zoff0 = g->nranks > 1 ? e0->z0 : 0;
  for (auto& e : t->eng) {
    const size_t off = (size_t)(e->z0 - zoff0) * e->Pr.g.plane;
    copy_in(e.get(), (const T*)m + off, const_cast<T*>(e->Pr.m), (size_t)e->Pr.g.N);
  }
  t->solve(g->opt, max_iter, eps_feas, eps_evol_of(g, tol), 1, 1, nullptr, nullptr);
  for (auto& e : t->eng) {
    const size_t off = (size_t)(e->z0 - zoff0) * e->Pr.g.plane;
    copy_out(e.get(), e->Pr.x, (T*)x + off, (size_t)e->Pr.g.N);
  }
  CU(cudaEventRecord(e0->ev1, g->stream));
  CU(cudaEventSynchronize(e0->ev1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0->ev0, e0->ev1);
  e0->fill_result(res, ms);
  g->have_m = true;
  g->last_launches = t->launches;
  g->last = e0;
  g->last_team = t;
  for (auto& e : t->eng)
    if (e->hc.numeric_err) throw SipError{SIP_ERR_NUMERIC, "NaN/Inf in the PARSDMM state"};
  return e0->hc.converged ? SIP_OK : SIP_NOT_CONVERGED;
}

template <class T>
sip_status project_T(sip_grid g, const void* m, void* x, int max_iter, double tol, sip_result* res) {
  if (is_team(g)) return project_team_T<T>(g, m, x, max_iter, tol, res);
  Engine<T>* e = engine_of<T>(g);
  const size_t N = (size_t)e->Pr.g.N;
  const double eps_feas = tol > 0 ? tol : 1e-3;
  e->launches = 0;
  e->prof = g->opt.profile != 0;
  for (int q = 0; q < Engine<T>::NKIND; ++q) { e->prof_ms[q] = 0; e->prof_cnt[q] = 0; }
  CU(cudaEventRecord(e->ev0, e->stream));
  copy_in(e, m, const_cast<T*>(e->Pr.m), N);
  const bool warm = g->opt.warm_start && e->ran && !e->scratch_used;
  if (warm) {
    e->rotate_final_to_read();
    std::vector<double> rho(e->hc.rho, e->hc.rho + e->P), gam(e->hc.gamma, e->hc.gamma + e->P);
    e->solve(g->opt, max_iter, eps_feas, eps_evol_of(g, tol), 0, 0, rho.data(), gam.data());
  } else {
    e->solve(g->opt, max_iter, eps_feas, eps_evol_of(g, tol), 1, 1, nullptr, nullptr);
  }
  copy_out(e, e->Pr.x, x, N);
  CU(cudaEventRecord(e->ev1, e->stream));
  CU(cudaEventSynchronize(e->ev1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e->ev0, e->ev1);
  e->fill_result(res, ms);
  g->have_m = true;
  g->last_launches = e->launches;
  g->last = e;
  if (e->hc.numeric_err) throw SipError{SIP_ERR_NUMERIC, e->hc.numeric_err == 3 ? "internal: kernel variant does not match the iteration" : e->hc.numeric_err == 4 ? "internal: threshold search window inconsistent" : "NaN/Inf in the PARSDMM state"};
  return e->hc.converged ? SIP_OK : SIP_NOT_CONVERGED;
}

template <class T>
sip_status multilevel_T(sip_grid g, const void* m, void* x, int n_levels, int max_iter, double tol,
                        sip_result* per_level) {
  // level grids: each axis halves (y stays 1 in 2D), h doubles (reading L2)
  if ((int)g->levels.size() != n_levels) {
    g->levels.clear();
    g->last = nullptr; g->last_team = nullptr;
    for (int l = 0; l < n_levels; ++l) {
      auto e = std::make_unique<Engine<T>>();
      const int f = 1 << l;
      double hl[3] = {g->h[0] * f, g->ndim == 3 ? g->h[1] * f : 1.0, g->h[2] * f};
      e->setup(g->ndim, (int)(g->n[0] / f), g->ndim == 3 ? (int)(g->n[1] / f) : 1, (int)(g->n[2] / f),
               hl, g->stream, g->sets);
      g->levels.push_back(std::move(e));
    }
  }
  auto L = [&](int l) { return static_cast<Engine<T>*>(g->levels[l].get()); };
  Engine<T>* fine = L(0);
  const size_t N = (size_t)fine->Pr.g.N;
  const double eps_feas = tol > 0 ? tol : 1e-3;
  CU(cudaEventRecord(fine->ev0, g->stream));
  copy_in(fine, m, const_cast<T*>(fine->Pr.m), N);
  for (int l = 1; l < n_levels; ++l) {
    k_restrict<T><<<L(l)->g_small_(), BLOCK, 0, g->stream>>>(L(l - 1)->Pr.g, L(l)->Pr.g, L(l - 1)->Pr.m,
                                                          const_cast<T*>(L(l)->Pr.m));
  }
  CU(cudaGetLastError());
  long long launches = n_levels - 1;
  std::vector<double> rho, gam;
  for (int l = n_levels - 1; l >= 0; --l) {
    Engine<T>* e = L(l);
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a)); CU(cudaEventCreate(&b));
    CU(cudaEventRecord(a, g->stream));
    e->launches = 0;
    e->prof = g->opt.profile != 0;   // per-kernel profile of every level (sip_get_profile: the finest)
    for (int q = 0; q < Engine<T>::NKIND; ++q) { e->prof_ms[q] = 0; e->prof_cnt[q] = 0; }
    if (l == n_levels - 1) {
      // coarsest: x = m_L, y_i = v_i = 0 (reading L13)
      for (int i = 0; i < e->P; ++i) {
        SetD<T>& S = e->Pr.set[i];
        CU(cudaMemsetAsync(S.y[1] - (size_t)GHOST * e->Pr.g.plane, 0, (size_t)S.nblk * e->Pr.g.ld * sizeof(T), g->stream));
        CU(cudaMemsetAsync(S.v[1] - (size_t)GHOST * e->Pr.g.plane, 0, (size_t)S.nblk * e->Pr.g.ld * sizeof(T), g->stream));
      }
      e->solve(g->opt, max_iter, eps_feas, eps_evol_of(g, tol), 1, 0, nullptr, nullptr);
    } else {
      Engine<T>* c = L(l + 1);
      // prolong x, y_i, v_i of the coarse level's final state (Algorithm 3)
      const int gs = e->g_small_();
      k_prolong<T><<<gs, BLOCK, 0, g->stream>>>(e->Pr.g, c->Pr.g, PRIM_I, c->Pr.x, e->Pr.x);
      e->launches++;
      for (int i = 0; i < e->P; ++i) {
        const SetD<T>& Sc = c->Pr.set[i];
        SetD<T>& Sf = e->Pr.set[i];
        const T* yc = c->final_field(i, 0);
        const T* vc = c->final_field(i, 1);
        for (int bl = 0; bl < Sf.nblk; ++bl) {
          k_prolong<T><<<gs, BLOCK, 0, g->stream>>>(e->Pr.g, c->Pr.g, Sf.prim[bl], yc + (int64_t)bl * c->Pr.g.ld,
                                                    Sf.y[1] + (int64_t)bl * e->Pr.g.ld);
          k_prolong<T><<<gs, BLOCK, 0, g->stream>>>(e->Pr.g, c->Pr.g, Sf.prim[bl], vc + (int64_t)bl * c->Pr.g.ld,
                                                    Sf.v[1] + (int64_t)bl * e->Pr.g.ld);
          e->launches += 2;
        }
        (void)Sc;
      }
      CU(cudaGetLastError());
      e->solve(g->opt, max_iter, eps_feas, eps_evol_of(g, tol), 0, 0, rho.data(), gam.data());
    }
    rho.assign(e->hc.rho, e->hc.rho + e->P);   // rho, gamma carry over (L23)
    gam.assign(e->hc.gamma, e->hc.gamma + e->P);
    CU(cudaEventRecord(b, g->stream));
    CU(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a); cudaEventDestroy(b);
    if (per_level) e->fill_result(&per_level[l], ms);
    launches += e->launches;
    if (e->hc.numeric_err) throw SipError{SIP_ERR_NUMERIC, e->hc.numeric_err == 3 ? "internal: kernel variant does not match the iteration" : e->hc.numeric_err == 4 ? "internal: threshold search window inconsistent" : "NaN/Inf in the PARSDMM state"};
  }
  copy_out(fine, fine->Pr.x, x, N);
  CU(cudaStreamSynchronize(g->stream));
  g->last_launches = launches;
  g->last = fine;
  return fine->hc.converged ? SIP_OK : SIP_NOT_CONVERGED;
}

// Algorithm 3 on z slabs: every level is a Team of the same G ranks; the
// slabs of all levels nest (nz divisible by G 2^(L-1)), so the restriction
// is slab-local; the prolongation reads one coarse ghost plane on each side,
// filled by a halo exchange of the coarse level's final x, y_i, v_i.
template <class T>
sip_status multilevel_team_T(sip_grid g, const void* m, void* x, int n_levels, int max_iter, double tol,
                             sip_result* per_level) {
  const bool nc = g->nranks > 1;
  const int G = nc ? g->nranks : g->vranks;
  if (g->n[0] % ((int64_t)G << (n_levels - 1)) != 0)
    throw SipError{SIP_ERR_CONFIG, "multilevel on z slabs needs nz divisible by ranks * 2^(levels-1)"};
  if ((int)g->levels.size() != n_levels) {
    g->levels.clear();
    g->last = nullptr; g->last_team = nullptr;
    if (!nc && !g->comm) {
      auto lc = std::make_unique<LocalComm>();
      lc->G = G;
      g->comm = std::move(lc);
    }
    for (int l = 0; l < n_levels; ++l) {
      const int f = 1 << l;
      double hl[3] = {g->h[0] * f, g->ndim == 3 ? g->h[1] * f : 1.0, g->h[2] * f};
      auto t = std::make_unique<Team<T>>();
      t->setup(g->ndim, (int)(g->n[0] / f), g->ndim == 3 ? (int)(g->n[1] / f) : 1, (int)(g->n[2] / f), hl,
               g->stream, g->sets, G, nc ? g->rank : 0, nc ? 1 : G, g->comm.get());
      g->levels.push_back(std::move(t));
    }
  }
  auto L = [&](int l) { return static_cast<Team<T>*>(g->levels[l].get()); };
  Team<T>* fine = L(0);
  const double eps_feas = tol > 0 ? tol : 1e-3;
  Engine<T>* f0 = fine->eng[0].get();
  CU(cudaEventRecord(f0->ev0, g->stream));
  const int64_t zoff0 = nc ? f0->z0 : 0;
  for (auto& e : fine->eng)
    copy_in(e.get(), (const T*)m + (size_t)(e->z0 - zoff0) * e->Pr.g.plane, const_cast<T*>(e->Pr.m),
            (size_t)e->Pr.g.N);
  long long launches = 0;
  for (int l = 1; l < n_levels; ++l)
    for (size_t r = 0; r < fine->eng.size(); ++r) {
      Engine<T>* ef = L(l - 1)->eng[r].get();
      Engine<T>* ec = L(l)->eng[r].get();
      k_restrict<T><<<ec->g_small_(), BLOCK, 0, g->stream>>>(ef->Pr.g, ec->Pr.g, ef->Pr.m, const_cast<T*>(ec->Pr.m));
      ++launches;
    }
  CU(cudaGetLastError());
  std::vector<double> rho, gam;
  for (int l = n_levels - 1; l >= 0; --l) {
    Team<T>* t = L(l);
    Engine<T>* e0 = t->eng[0].get();
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a)); CU(cudaEventCreate(&b));
    CU(cudaEventRecord(a, g->stream));
    if (l == n_levels - 1) {
      for (auto& e : t->eng)   // coarsest: x = m_L, y_i = v_i = 0 (reading L13)
        for (int i = 0; i < e->P; ++i) {
          SetD<T>& S = e->Pr.set[i];
          CU(cudaMemsetAsync(S.y[1] - (size_t)GHOST * e->Pr.g.plane, 0, (size_t)S.nblk * e->Pr.g.ld * sizeof(T), g->stream));
          CU(cudaMemsetAsync(S.v[1] - (size_t)GHOST * e->Pr.g.plane, 0, (size_t)S.nblk * e->Pr.g.ld * sizeof(T), g->stream));
        }
      t->solve(g->opt, max_iter, eps_feas, eps_evol_of(g, tol), 1, 0, nullptr, nullptr);
    } else {
      Team<T>* c = L(l + 1);
      const int kk = std::min(c->eng[0]->hc.k, c->eng[0]->hc.opt.max_iter);
      const int par = (kk + 1) & 1;   // parity of the coarse level's final y, v
      c->site(ST_INIT, 0, 0, {{FS_X, 0, H_BOTH}, {par ? FS_Y1 : FS_Y0, SS_ALLBLK, H_BOTH},
                              {par ? FS_V1 : FS_V0, SS_ALLBLK, H_BOTH}}, false);
      for (size_t r = 0; r < t->eng.size(); ++r) {
        Engine<T>* e = t->eng[r].get();
        Engine<T>* ec = c->eng[r].get();
        const int gs = e->g_small_();
        k_prolong<T><<<gs, BLOCK, 0, g->stream>>>(e->Pr.g, ec->Pr.g, PRIM_I, ec->Pr.x, e->Pr.x);
        ++launches;
        for (int i = 0; i < e->P; ++i) {
          SetD<T>& Sf = e->Pr.set[i];
          const T* yc = ec->final_field(i, 0);
          const T* vc = ec->final_field(i, 1);
          for (int bl = 0; bl < Sf.nblk; ++bl) {
            k_prolong<T><<<gs, BLOCK, 0, g->stream>>>(e->Pr.g, ec->Pr.g, Sf.prim[bl], yc + (int64_t)bl * ec->Pr.g.ld,
                                                      Sf.y[1] + (int64_t)bl * e->Pr.g.ld);
            k_prolong<T><<<gs, BLOCK, 0, g->stream>>>(e->Pr.g, ec->Pr.g, Sf.prim[bl], vc + (int64_t)bl * ec->Pr.g.ld,
                                                      Sf.v[1] + (int64_t)bl * e->Pr.g.ld);
            launches += 2;
          }
        }
      }
      CU(cudaGetLastError());
      t->solve(g->opt, max_iter, eps_feas, eps_evol_of(g, tol), 0, 0, rho.data(), gam.data());
    }
    rho.assign(e0->hc.rho, e0->hc.rho + e0->P);   // rho, gamma carry over (L23)
    gam.assign(e0->hc.gamma, e0->hc.gamma + e0->P);
    CU(cudaEventRecord(b, g->stream));
    CU(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a); cudaEventDestroy(b);
    if (per_level) e0->fill_result(&per_level[l], ms);
    launches += t->launches;
    for (auto& e : t->eng)
      if (e->hc.numeric_err) throw SipError{SIP_ERR_NUMERIC, "NaN/Inf in the PARSDMM state"};
  }
  for (auto& e : fine->eng)
    copy_out(e.get(), e->Pr.x, (T*)x + (size_t)(e->z0 - zoff0) * e->Pr.g.plane, (size_t)e->Pr.g.N);
  CU(cudaStreamSynchronize(g->stream));
  g->last_launches = launches;
  g->last = f0;
  g->last_team = fine;
  return f0->hc.converged ? SIP_OK : SIP_NOT_CONVERGED;
}

template <class T>
sip_status apply_op_E(Engine<T>* e, int set_id, const void* x, void* y);
template <class T>
sip_status apply_op_T(sip_grid g, int set_id, const void* x, void* y) {
  return apply_op_E<T>(engine_of<T>(g), set_id, x, y);
}
template <class T>
sip_status apply_op_E(Engine<T>* e, int set_id, const void* x, void* y) {
  const Geo& G = e->Pr.g;
  const SetD<T>& S = e->Pr.set[set_id];
  T* xin = e->Pr.pb[0];
  copy_in(e, x, xin, G.N);
  T* out = e->Pr.hist[0];   // scratch: nblk blocks needed -> use hist slots
  T* tmp[3] = {e->Pr.hist[0], e->Pr.hist[1], e->Pr.hist[2]};
  (void)out;
  // k_apply_op writes block b at out + b*ld: use contiguous scratch of nblk*ld
  T* scratch = e->template dalloc<T>((size_t)S.nblk * G.ld);
  k_apply_op<T><<<e->g_small_(), BLOCK, 0, e->stream>>>(e->Pr, set_id, xin, scratch);
  const long long M = e->set_len(set_id);
  T* comp = e->template dalloc<T>(M);
  long long boff = 0;
  for (int b = 0; b < S.nblk; ++b) {
    k_pack<T, T><<<e->g_small_(), BLOCK, 0, e->stream>>>(G, S.prim[b], e->d_fmap, boff, scratch + (int64_t)b * G.ld, comp, 0);
    boff += e->block_len(S.prim[b]);
  }
  CU(cudaGetLastError());
  copy_out(e, comp, y, M);
  CU(cudaStreamSynchronize(e->stream));
  (void)tmp;
  // release the scratch (last two allocations)
  cudaFree(comp); e->allocs.pop_back();
  cudaFree(scratch); e->allocs.pop_back();
  return SIP_OK;
}

template <class T>
void set_rho_coeffs(Engine<T>* e, const double* rho) {
  Ctrl c = e->hc;
  for (int i = 0; i < e->P; ++i) c.rho[i] = rho[i];
  make_coeffs(e->Pr, c.rho, &c.cI, &c.cz, &c.cy, &c.cx, &c.cF);
  e->hc = c;
  CU(cudaMemcpyAsync(e->d_ctrl, &e->hc, sizeof(Ctrl), cudaMemcpyHostToDevice, e->stream));
}

template <class T>
sip_status apply_system_T(sip_grid g, const double* rho, const void* pin, void* qout) {
  Engine<T>* e = engine_of<T>(g);
  const Geo& G = e->Pr.g;
  set_rho_coeffs(e, rho);
  T* pv = e->Pr.pb[0];
  T* q = e->Pr.pb[1];
  copy_in(e, pin, pv, G.N);
  if (e->Pr.has[PRIM_F]) {
    // tb = S G p: reuse k_blur_t mode 0 on x := p
    Prob<T> P2 = e->Pr;
    P2.x = pv;
    Ctrl c = e->hc; c.stopped = 0;
    e->hc = c;
    CU(cudaMemcpyAsync(e->d_ctrl, &e->hc, sizeof(Ctrl), cudaMemcpyHostToDevice, e->stream));
    k_blur_t<T><<<e->g_pts, BLOCK, 0, e->stream>>>(P2, 0, 0);
  }
  k_apply_sys<T><<<e->g_small_(), BLOCK, 0, e->stream>>>(e->Pr, e->d_ctrl, pv, nullptr, q, 0);
  CU(cudaGetLastError());
  copy_out(e, q, qout, G.N);
  CU(cudaStreamSynchronize(e->stream));
  return SIP_OK;
}

template <class T>
sip_status cg_T(sip_grid g, const double* rho, const void* b, void* x, int n_cg, int eq25, int* iters) {
  Engine<T>* e = engine_of<T>(g);
  const Geo& G = e->Pr.g;
  // control block for a bare CG solve: Eq. 25 from r0 = b - C x
  e->ensure_log(1);
  const double floor_ = g->opt.cg_tol_floor > 0 ? g->opt.cg_tol_floor
                                                : 10.0 * (sizeof(T) == 4 ? (double)FLT_EPSILON : DBL_EPSILON);
  Options o = g->opt;
  o.n_cg = n_cg; o.eq25 = eq25;
  e->ensure_ring(n_cg);
  e->fill_ctrl(o, 1, 1e-3, 1e-2, floor_, rho, nullptr);
  T* bb = e->Pr.hist[1];
  copy_in(e, b, bb, G.N);
  copy_in(e, x, e->Pr.x, G.N);
  // r = b - C x and the CG flags: run k_rhs on a problem whose right-hand
  // side is b, i.e. rho_i y_i + v_i replaced: use a 1-set identity view
  Prob<T> P2 = e->Pr;
  P2.P = 1;   // only the distance block contributes to b: rho*y + v with y = b/rho, v = 0
  P2.set[0] = e->Pr.set[e->P - 1];
  P2.set[0].y[0] = P2.set[0].y[1] = bb;
  T* zero = e->Pr.hist[2];
  CU(cudaMemsetAsync(zero, 0, G.N * sizeof(T), e->stream));
  P2.set[0].v[0] = P2.set[0].v[1] = zero;
  // scale: k_rhs computes rho_{P2.set0} * y + v with rho = C.rho[0]; set rho[0] = 1 in a copy
  Ctrl c = e->hc;
  c.rho[0] = 1.0;   // coefficient of b (the C coefficients keep the caller's rho)
  e->hc = c;
  CU(cudaMemcpyAsync(e->d_ctrl, &e->hc, sizeof(Ctrl), cudaMemcpyHostToDevice, e->stream));
  if (e->Pr.has[PRIM_F]) { k_blur_t<T><<<e->g_pts, BLOCK, 0, e->stream>>>(P2, 0, 0); }
  k_rhs<T><<<e->g_pts, BLOCK, 0, e->stream>>>(P2);
  for (int j = 0; j < n_cg; ++j) {
    if (e->lean_cg()) {   // the same kernels as the hot path
      if (e->Pr.has[PRIM_F]) k_blurF<T><<<e->g_bf, BLOCK, e->smem_bf, e->stream>>>(e->Pr, j);
      e->launch_cg1(j);
      e->launch_cg2(j);
    } else {
      if (e->Pr.has[PRIM_F]) k_blur_t<T><<<e->g_pts, BLOCK, 0, e->stream>>>(e->Pr, 1, j);
      k_cg1<T><<<e->g_pts, BLOCK, 0, e->stream>>>(e->Pr, j);
      k_cg2<T><<<e->g_pts, BLOCK, 0, e->stream>>>(e->Pr, j);
    }
  }
  if (e->Pr.defer_x && n_cg > 0) e->launch_cgx();
  CU(cudaGetLastError());
  e->read_ctrl();
  copy_out(e, e->Pr.x, x, G.N);
  CU(cudaStreamSynchronize(e->stream));
  if (iters) *iters = e->hc.cg_count;
  return SIP_OK;
}

template <class T>
sip_status project_set_E(Engine<T>* e, int set_id, const void* w, void* y);
template <class T>
sip_status project_set_T(sip_grid g, int set_id, const void* w, void* y) {
  Engine<T>* e = engine_of<T>(g);
  if (!e->ran) throw SipError{SIP_ERR_STATE, "sip_project_set needs a previous sip_project"};
  return project_set_E<T>(e, set_id, w, y);
}
template <class T>
sip_status project_set_E(Engine<T>* e, int set_id, const void* w, void* y) {
  // the step-level projection runs pass 1 / the radix rounds directly (no
  // select v2: its round-A counts would be left behind for the next solve)
  struct V2Off {
    int* f; int v;
    ~V2Off() { *f = v; }
  } v2off{&e->Pr.selv2, e->Pr.selv2};
  e->Pr.selv2 = 0;
  const Geo& G = e->Pr.g;
  SetD<T>& S = e->Pr.set[set_id];
  const long long M = e->set_len(set_id);
  T* comp = e->template dalloc<T>(M);
  copy_in(e, w, comp, M);
  // Run the hot-path kernels on a control block for iteration k = 2 (no
  // adapt, no check): pass1 reads y[0]/v[0] and writes y[1]/v[1]; pass2
  // writes y[1].  Only this set's select job is active.  The grid's state
  // buffers are used as scratch (a later warm start is refused).
  Ctrl c = e->hc;
  c.k = 2; c.stopped = 0; c.first_adapt_done = 0; c.adapt_calls = 0;
  c.opt.check_every = 1 << 30;
  c.opt.adapt_every = 2;
  for (int i = 0; i < e->P; ++i) { c.rho[i] = 1.0; c.gamma[i] = 1.0; }
  for (int jb = 0; jb < c.njobs; ++jb) {
    Job& J = c.job[jb];
    const int i = J.set;
    J.round = 0; J.prefix = 0; J.cnt_above = 0; J.sum_above = 0; J.theta = 0; J.tau = 0;
    J.keep_eq = 0; J.cnt_eq = 0; J.ties = 0; J.tau_val2 = 0; J.cand_n = 0;
    J.sigma = c.sigma[i]; J.k = c.kcard[i];
    J.mode = (J.on_s || i != set_id) ? JM_OFF : JM_SEARCH;
    if (J.mode == JM_SEARCH && J.kind == K_CARD) {
      if (J.k <= 0) J.mode = JM_ZERO;
      else if (J.k >= c.mreal[i]) J.mode = JM_ALL;
    }
  }
  if (S.global) {
    long long boff = 0;
    for (int b = 0; b < S.nblk; ++b) {
      k_pack<T, T><<<e->g_small_(), BLOCK, 0, e->stream>>>(G, S.prim[b], e->d_fmap, boff,
                                                           S.w + (int64_t)b * G.ld, comp, 1);
      boff += e->block_len(S.prim[b]);
    }
    if (S.kind == K_L2 || S.kind == K_ANN) {
      // the radial factor comes from pass1's ||w||^2 in the hot path; here w
      // is given, so its norm is formed on the host (step-level entry only)
      std::vector<T> hw(M);
      copy_out(e, comp, hw.data(), M);
      CU(cudaStreamSynchronize(e->stream));
      double w2 = 0.0;
      for (long long q = 0; q < M; ++q) w2 += (double)hw[q] * (double)hw[q];
      const double n = std::sqrt(w2);
      double f = 1.0; int z = 0;
      if (n == 0.0) z = c.sig_lo[set_id] > 0.0;
      else if (n > c.sig_hi[set_id]) f = c.sig_hi[set_id] / n;
      else if (n < c.sig_lo[set_id]) f = c.sig_lo[set_id] / n;
      c.ann_scale[set_id] = f; c.ann_zero[set_id] = z;
    }
    e->hc = c;
    CU(cudaMemcpyAsync(e->d_ctrl, &e->hc, sizeof(Ctrl), cudaMemcpyHostToDevice, e->stream));
    if (S.dct) e->dct_field(S.w, 0, S.dct);   // the search and pass 2 act on D w
    if (S.svd) {   // rank / nuclear-norm set: the batched Jacobi kernel writes y[1]
      const MatView mv = mat_view(e->ndim, e->nz_g, e->ny, e->nx, S.prim[0]);
      e->launch_svd_one(set_id, 0, mv.nmat);
    } else if (S.fib) {   // per-fiber projection: k_fiberw / k_fiber write y[1]
      if (S.fpath) FiberW<T>::of(S.flen)<<<e->g_fw[set_id], BLOCK, e->smem_fw[set_id], e->stream>>>(e->Pr, set_id);
      else k_fiber<T><<<e->g_fib, BLOCK, e->smem_fib, e->stream>>>(e->Pr);
    } else if (S.job >= 0) {
      for (int r = 1; r <= KeyT<T>::ROUNDS; ++r) {
        if (e->vec) e->launch_select(r);
        else k_select<T><<<e->g_sel, BLOCK, 0, e->stream>>>(e->Pr, r);
      }
      if (S.kind == K_CARD) {
        if (e->vec) k_tiecountf<T><<<e->g_p2, BLOCK, 0, e->stream>>>(e->Pr);
        else k_tiecount<T><<<e->g_p2, BLOCK, 0, e->stream>>>(e->Pr);
      }
    }
    if (S.fib || S.svd) {
    } else if (e->vec) k_pass2t<T, 2, 2><<<e->g_p2, BLOCK, e->smem_p2, e->stream>>>(e->Pr);
    else k_pass2<T><<<e->g_p2, BLOCK, e->smem_p2, e->stream>>>(e->Pr);
    if (S.dct) e->dct_field(S.y[1], 1, S.dct);   // y = D^T P_l1(D w)
  } else {
    // pointwise: gamma = 0 and v = 0 make x-bar = y_old and w = y_old, so
    // pass1 evaluates y = P(w) on the given w placed in y[0]
    c.gamma[set_id] = 0.0;
    e->hc = c;
    CU(cudaMemcpyAsync(e->d_ctrl, &e->hc, sizeof(Ctrl), cudaMemcpyHostToDevice, e->stream));
    long long boff = 0;
    for (int b = 0; b < S.nblk; ++b) {
      k_pack<T, T><<<e->g_small_(), BLOCK, 0, e->stream>>>(G, S.prim[b], e->d_fmap, boff,
                                                           S.y[0] + (int64_t)b * G.ld, comp, 1);
      CU(cudaMemsetAsync(S.v[0] + (int64_t)b * G.ld, 0, G.N * sizeof(T), e->stream));
      boff += e->block_len(S.prim[b]);
    }
    if (e->vec) k_pass1t<T, 2, 2><<<e->g_p1a, BLOCK, e->smem_p1a, e->stream>>>(e->Pr);
    else k_pass1<T><<<e->g_pts, BLOCK, e->smem_p1, e->stream>>>(e->Pr);
  }
  CU(cudaGetLastError());
  long long boff = 0;
  for (int b = 0; b < S.nblk; ++b) {
    k_pack<T, T><<<e->g_small_(), BLOCK, 0, e->stream>>>(G, S.prim[b], e->d_fmap, boff,
                                                         S.y[1] + (int64_t)b * G.ld, comp, 0);
    boff += e->block_len(S.prim[b]);
  }
  copy_out(e, comp, y, M);
  CU(cudaStreamSynchronize(e->stream));
  cudaFree(comp); e->allocs.pop_back();
  e->ran = false;
  e->read_ctrl();
  e->ran = true;      // parameters (sigma, k) stay resolved; state is scratch
  e->scratch_used = true;
  return SIP_OK;
}

template <class T>
Engine<T>* last_engine(sip_grid g) {
  return g->last ? static_cast<Engine<T>*>(g->last) : engine_of<T>(g);
}

template <class T>
sip_status get_state_T(sip_grid g, int set_id, int which, void* out) {
  Engine<T>* e = last_engine<T>(g);
  if (!e->ran) throw SipError{SIP_ERR_STATE, "no projection state"};
  const Geo& G = e->Pr.g;
  const SetD<T>& S = e->Pr.set[set_id];
  const long long M = (set_id == e->p) ? G.N : e->set_len(set_id);
  T* src = e->final_field(set_id, which);
  T* comp = e->template dalloc<T>(M);
  long long boff = 0;
  for (int b = 0; b < S.nblk; ++b) {
    k_pack<T, T><<<e->g_small_(), BLOCK, 0, e->stream>>>(G, S.prim[b], e->d_fmap, boff, src + (int64_t)b * G.ld, comp, 0);
    boff += e->block_len(S.prim[b]);
  }
  CU(cudaGetLastError());
  copy_out(e, comp, out, M);
  CU(cudaStreamSynchronize(e->stream));
  cudaFree(comp); e->allocs.pop_back();
  return SIP_OK;
}

// z slabs: the compact field of set i, block-major, each block the slabs of
// this process's ranks in rank order (virtual ranks: the whole field)
template <class T>
sip_status get_state_team_T(sip_grid g, int set_id, int which, void* out) {
  Team<T>* t = static_cast<Team<T>*>(g->last_team);
  if (!t || !t->ran) throw SipError{SIP_ERR_STATE, "no projection state"};
  const SetD<T>& S0 = t->eng[0]->Pr.set[set_id];
  long long off = 0;
  for (int b = 0; b < S0.nblk; ++b)
    for (auto& e : t->eng) {
      const Geo& G = e->Pr.g;
      const long long len = e->block_len(S0.prim[b]);
      T* comp = e->template dalloc<T>((size_t)std::max(len, 1ll));
      T* src = e->final_field(set_id, which) + (int64_t)b * G.ld;
      k_pack<T, T><<<e->g_small_(), BLOCK, 0, e->stream>>>(G, S0.prim[b], e->d_fmap, 0, src, comp, 0);
      CU(cudaGetLastError());
      copy_out(e.get(), comp, (T*)out + off, (size_t)len);
      CU(cudaStreamSynchronize(e->stream));
      cudaFree(comp); e->allocs.pop_back();
      off += len;
    }
  return SIP_OK;
}

template <class T>
sip_status get_log_T(sip_grid g, int max_iter, int* cg, int* branch, double* rho_t, double* gam_t,
                     double* feas, double* evol) {
  Engine<T>* e = last_engine<T>(g);
  if (!e->ran) throw SipError{SIP_ERR_STATE, "no projection log"};
  const int n = std::min(max_iter, e->log_cap);
  const int P = e->P, p = e->p;
  if (cg) CU(cudaMemcpy(cg, e->d_log_cg, n * sizeof(int), cudaMemcpyDeviceToHost));
  if (branch) CU(cudaMemcpy(branch, e->d_log_br, (size_t)n * P * sizeof(int), cudaMemcpyDeviceToHost));
  if (rho_t) CU(cudaMemcpy(rho_t, e->d_log_rho, (size_t)n * P * sizeof(double), cudaMemcpyDeviceToHost));
  if (gam_t) CU(cudaMemcpy(gam_t, e->d_log_gam, (size_t)n * P * sizeof(double), cudaMemcpyDeviceToHost));
  if (feas && p) CU(cudaMemcpy(feas, e->d_log_feas, (size_t)n * p * sizeof(double), cudaMemcpyDeviceToHost));
  if (evol) CU(cudaMemcpy(evol, e->d_log_evol, n * sizeof(double), cudaMemcpyDeviceToHost));
  return SIP_OK;
}

// ---- Algorithm 4, parallel Dykstra: the Fig. 1 comparator --
// Sub-problem i (P_{V_i}): the set's projector when A_i = I, else PARSDMM
// with that one set (the paper's ARADMM role) on an engine of its own,
// started from v_i; relative parameters resolved once from m by the main
// engine; weights 1/p; counters of P:497-501 per outer iteration.
struct DykState : EngineBase {
  std::vector<std::vector<HostSet>> sets;       // one set per sub-engine (absolute parameters)
  std::vector<std::unique_ptr<EngineBase>> eng;
};

template <class T>
sip_status dykstra_T(sip_grid g, const void* m_in, void* x_out, int max_outer, double tol, int inner_max,
                     double inner_tol, sip_dykstra_log* log) {
  if (is_team(g)) throw SipError{SIP_ERR_CONFIG, "sip_dykstra: one rank only"};
  Engine<T>* e = engine_of<T>(g);
  const int p = e->p;
  if (p < 1) throw SipError{SIP_ERR_CONFIG, "sip_dykstra needs at least one set"};
  const size_t N = (size_t)e->Pr.g.N;
  // resolve the relative parameters from m: one iteration of the main engine
  copy_in(e, m_in, const_cast<T*>(e->Pr.m), N);
  e->solve(g->opt, 1, 1e-3, 1e-2, 1, 1, nullptr, nullptr);
  auto st = std::make_unique<DykState>();
  for (int i = 0; i < p; ++i) {
    HostSet hs = g->sets[i];
    hs.prm.relative = 0;
    hs.prm.sigma = e->hc.sigma[i];
    hs.prm.sigma_lo = e->hc.sig_lo[i];
    hs.prm.sigma_hi = e->hc.sig_hi[i];
    hs.prm.k = e->hc.kcard[i];
    if (hs.type == SIP_SET_L2_BALL) hs.prm.sigma = e->hc.sig_hi[i];
    st->sets.push_back({hs});
  }
  for (int i = 0; i < p; ++i) {
    auto se = std::make_unique<Engine<T>>();
    se->setup(g->ndim, (int)g->n[0], (int)g->n[1], (int)g->n[2], g->h, g->stream, st->sets[i]);
    st->eng.push_back(std::move(se));
  }
  auto E = [&](int i) { return static_cast<Engine<T>*>(st->eng[i].get()); };
  struct Release {   // this call's work buffers: freed on return (e->allocs is append-only)
    Engine<T>* e; size_t n0;
    ~Release() { while (e->allocs.size() > n0) { cudaFree(e->allocs.back()); e->allocs.pop_back(); } }
  } rel{e, e->allocs.size()};
  T* x = e->template dalloc<T>(N);
  T* xo = e->template dalloc<T>(N);
  DykPtrs<T> ptr{};
  for (int i = 0; i < p; ++i) { ptr.y[i] = e->template dalloc<T>(N); ptr.v[i] = e->template dalloc<T>(N); }
  long long Mmax = (long long)N;
  for (int i = 0; i < p; ++i) Mmax = std::max(Mmax, E(i)->set_len(0));
  T* a = e->template dalloc<T>((size_t)Mmax);
  T* pa = e->template dalloc<T>((size_t)Mmax);
  double* red = e->template dalloc<double>(2);
  copy_in(e, m_in, x, N);                                                   // 0a
  for (int i = 0; i < p; ++i)                                               // 0b
    CU(cudaMemcpyAsync(ptr.v[i], x, N * sizeof(T), cudaMemcpyDeviceToDevice, g->stream));
  Options oin = g->opt;                                                     // the sub-problems: natural mode
  oin.fixed_work = 0;
  oin.eq25 = 1;
  const double eps_evol = inner_tol > 0 ? 10.0 * inner_tol : 1e-2;
  int k;
  double h2[2];
  for (k = 1; k <= max_outer; ++k) {
    int cg_max = 0, l1p = 0;
    for (int i = 0; i < p; ++i) {                                           // 1: y_i = P_{V_i}(v_i)
      Engine<T>* s = E(i);
      int it = 0, cg = 0;
      if (st->sets[i][0].op == SIP_OP_IDENTITY) {
        if (!s->ran) { copy_in(s, ptr.v[i], const_cast<T*>(s->Pr.m), N); s->solve(oin, 1, 1e-3, 1e-2, 1, 1, nullptr, nullptr); }
        project_set_E<T>(s, 0, ptr.v[i], ptr.y[i]);
        it = 1;
      } else {
        CU(cudaMemcpyAsync(const_cast<T*>(s->Pr.m), ptr.v[i], N * sizeof(T), cudaMemcpyDeviceToDevice, g->stream));
        s->solve(oin, inner_max, inner_tol > 0 ? inner_tol : 1e-3, eps_evol, 1, 1, nullptr, nullptr);
        CU(cudaMemcpyAsync(ptr.y[i], s->Pr.x, N * sizeof(T), cudaMemcpyDeviceToDevice, g->stream));
        it = std::min(s->hc.k, s->hc.opt.max_iter);
        cg = s->hc.cg_total;
      }
      cg_max = std::max(cg_max, cg);
      if (st->sets[i][0].type == SIP_SET_L1_BALL) l1p += it;
      if (log && log->inner_iters) log->inner_iters[(size_t)(k - 1) * p + i] = it;
    }
    k_dyk_update<T><<<e->g_small_(), BLOCK, 0, g->stream>>>(x, xo, ptr, p, (long long)N, e->Pr.partials,
                                                             e->Pr.counter, red);          // 2, 3
    CU(cudaMemcpyAsync(h2, red, 2 * sizeof(double), cudaMemcpyDeviceToHost, g->stream));
    CU(cudaStreamSynchronize(g->stream));
    const double re = h2[1] > 0.0 ? std::sqrt(h2[0]) / std::sqrt(h2[1]) : 0.0;
    if (log) {
      if (log->cg_max) log->cg_max[k - 1] = cg_max;
      if (log->l1_proj) log->l1_proj[k - 1] = l1p;
      if (log->r_evol) log->r_evol[k - 1] = re;
      if (log->r_feas)
        for (int i = 0; i < p; ++i) {                                       // Eq. 26 of x^k
          Engine<T>* s = E(i);
          const long long M = s->set_len(0);
          apply_op_E<T>(s, 0, x, a);
          project_set_E<T>(s, 0, a, pa);
          k_feas2<T><<<e->g_small_(), BLOCK, 0, g->stream>>>(a, pa, M, e->Pr.partials, e->Pr.counter, red);
          CU(cudaMemcpyAsync(h2, red, 2 * sizeof(double), cudaMemcpyDeviceToHost, g->stream));
          CU(cudaStreamSynchronize(g->stream));
          log->r_feas[(size_t)(k - 1) * p + i] = h2[1] > 0.0 ? std::sqrt(h2[0]) / std::sqrt(h2[1]) : 0.0;
        }
    }
    if (re < tol) break;
  }
  if (log) log->iterations = k > max_outer ? max_outer : k;
  copy_out(e, x, x_out, N);
  CU(cudaStreamSynchronize(g->stream));
  g->dyk = std::move(st);
  return k > max_outer ? SIP_NOT_CONVERGED : SIP_OK;
}

template <class F>
sip_status guarded(sip_grid g, F&& f) {
  try {
    int cur;
    if (g && cudaGetDevice(&cur) == cudaSuccess && cur != g->device) cudaSetDevice(g->device);
    if (g && g->fence) {   // order the library stream after the caller's stream
      CU(cudaEventRecord(g->fence, g->user_stream));
      CU(cudaStreamWaitEvent(g->stream, g->fence, 0));
    }
    return f();
  } catch (const SipError& e) {
    if (g) g->err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    if (g) g->err = "host allocation failed";
    return SIP_ERR_OOM;
  }
}

}  // namespace

// ------------------------------------------------------------------ C ABI
extern "C" {

const char* sip_status_string(sip_status s) {
  switch (s) {
    case SIP_OK: return "ok";
    case SIP_NOT_CONVERGED: return "not converged (max_iter reached)";
    case SIP_ERR_ARG: return "invalid argument";
    case SIP_ERR_CONFIG: return "unsupported configuration";
    case SIP_ERR_PARAM: return "invalid set parameter";
    case SIP_ERR_SHAPE: return "shape mismatch";
    case SIP_ERR_CUDA: return "CUDA error";
    case SIP_ERR_NCCL: return "NCCL error";
    case SIP_ERR_OOM: return "out of memory";
    case SIP_ERR_NUMERIC: return "numerical failure (NaN/Inf)";
    case SIP_ERR_STATE: return "call out of order";
  }
  return "unknown status";
}

const char* sip_last_error(sip_grid g) { return g ? g->err.c_str() : "null grid"; }

sip_status sip_comm_unique_id(uint8_t out[128]) {
  if (!out) return SIP_ERR_ARG;
  memset(out, 0, 128);
  NcclApi& A = nccl();
  if (!A.ok) return SIP_ERR_NCCL;
  nccl_uid id;
  if (A.GetUniqueId(&id) != 0) return SIP_ERR_NCCL;
  memcpy(out, id.internal, 128);
  return SIP_OK;
}

sip_status sip_slab(int64_t nz, int nranks, int rank, int64_t* z0, int64_t* nz_local) {
  if (nz < 1 || nranks < 1 || rank < 0 || rank >= nranks || !z0 || !nz_local) return SIP_ERR_ARG;
  int a, b;
  slab_of((int)nz, nranks, rank, &a, &b);
  *z0 = a;
  *nz_local = b;
  return SIP_OK;
}

sip_status sip_create_grid(int ndim, const int64_t* n, const double* h, sip_dtype dtype,
                           const sip_comm_desc* comm, void* cuda_stream, sip_grid* out) {
  if (!out || !n || (ndim != 2 && ndim != 3) || (dtype != SIP_F32 && dtype != SIP_F64)) return SIP_ERR_ARG;
  *out = nullptr;
  for (int a = 0; a < ndim; ++a) if (n[a] < 2) return SIP_ERR_SHAPE;
  if (h) for (int a = 0; a < ndim; ++a) if (!(h[a] > 0)) return SIP_ERR_PARAM;
  if (comm && (comm->nranks < 1 || comm->rank < 0 || comm->rank >= comm->nranks)) return SIP_ERR_ARG;
  if (comm && comm->nranks > 1 && (!comm->nccl_unique_id || n[0] < comm->nranks)) return SIP_ERR_ARG;
  int64_t N = 1;
  for (int a = 0; a < ndim; ++a) N *= n[a];
  if (N >= (1ll << 31) - 8) return SIP_ERR_SHAPE;
  auto g = new (std::nothrow) sip_grid_s();
  if (!g) return SIP_ERR_OOM;
  if (cudaGetDevice(&g->device) != cudaSuccess) { cudaGetLastError(); delete g; return SIP_ERR_CUDA; }
  g->user_stream = (cudaStream_t)cuda_stream;
  if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&g->fence, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    delete g;
    return SIP_ERR_CUDA;
  }
  g->dtype = dtype;
  g->ndim = ndim;
  if (ndim == 2) {
    g->n[0] = n[0]; g->n[1] = 1; g->n[2] = n[1];
    g->h[0] = h ? h[0] : 1.0; g->h[1] = 1.0; g->h[2] = h ? h[1] : 1.0;
  } else {
    for (int a = 0; a < 3; ++a) { g->n[a] = n[a]; g->h[a] = h ? h[a] : 1.0; }
  }
  if (comm && comm->nranks > 1) {
    NcclApi& A = nccl();
    if (!A.ok) { delete g; return SIP_ERR_NCCL; }
    auto nc = std::make_unique<NcclComm>();
    nc->G = comm->nranks;
    nc->rank = comm->rank;
    nccl_uid id;
    memcpy(id.internal, comm->nccl_unique_id, 128);
    if (A.CommInitRank(&nc->comm, comm->nranks, id, comm->rank) != 0) { delete g; return SIP_ERR_NCCL; }
    g->nranks = comm->nranks;
    g->rank = comm->rank;
    g->comm = std::move(nc);
  }
  *out = g;
  return SIP_OK;
}

sip_status sip_add_set(sip_grid g, sip_op op, const void* op_desc, sip_set_type type,
                       const sip_set_params* prm, int* set_id) {
  if (!g || !prm) return SIP_ERR_ARG;
  if (op < SIP_OP_IDENTITY || op > SIP_OP_BLUR_MASK || type < SIP_SET_BOUNDS || type > SIP_SET_HAAR_L1)
    return SIP_ERR_ARG;
  if ((int)g->sets.size() >= SIP_MAX_SETS) { g->err = "more than 16 sets"; return SIP_ERR_CONFIG; }
  if (op == SIP_OP_DY && g->ndim != 3) { g->err = "D_y needs a 3D grid"; return SIP_ERR_CONFIG; }
  return guarded(g, [&]() -> sip_status {
    HostSet hs;
    hs.op = op; hs.type = type; hs.prm = *prm;
    hs.prm.lo_vec = hs.prm.hi_vec = nullptr;
    const int64_t N = g->n[0] * g->n[1] * g->n[2];
    const int64_t nz = g->n[0], ny = g->n[1], nx = g->n[2];
    if (op == SIP_OP_BLUR_MASK) {
      const sip_blur_mask_desc* d = (const sip_blur_mask_desc*)op_desc;
      if (!d || !d->kernel || !d->mask) return SIP_ERR_ARG;
      if (g->ndim != 2) { g->err = "blur/mask operator is 2D only"; return SIP_ERR_CONFIG; }
      if (d->kh < 1 || d->kw < 1 || d->kh % 2 == 0 || d->kw % 2 == 0 || d->kh > 9 || d->kw > 9 ||
          d->kh / 2 > GHOST * 2 || d->kw / 2 > 4) return SIP_ERR_PARAM;
      for (auto& s2 : g->sets) if (s2.op == SIP_OP_BLUR_MASK) { g->err = "one blur/mask operator per grid"; return SIP_ERR_CONFIG; }
      hs.kernel.assign(d->kernel, d->kernel + d->kh * d->kw);
      hs.kh = d->kh; hs.kw = d->kw;
      hs.mask.resize(N);
      if (is_device_ptr(d->mask)) CU(cudaMemcpy(hs.mask.data(), d->mask, N, cudaMemcpyDeviceToHost));
      else memcpy(hs.mask.data(), d->mask, N);
      int64_t c = 0;
      for (int64_t q = 0; q < N; ++q) c += hs.mask[q] ? 1 : 0;
      hs.M = c;
    } else {
      switch (op) {
        case SIP_OP_IDENTITY: hs.M = N; break;
        case SIP_OP_DZ: hs.M = (nz - 1) * ny * nx; break;
        case SIP_OP_DY: hs.M = nz * (ny - 1) * nx; break;
        case SIP_OP_DX: hs.M = nz * ny * (nx - 1); break;
        default: hs.M = (nz - 1) * ny * nx + (g->ndim == 3 ? nz * (ny - 1) * nx : 0) + nz * ny * (nx - 1);
      }
    }
    // parameter checks
    if (type == SIP_SET_BOUNDS) {
      if (!prm->lo_vec && !prm->hi_vec && !(prm->lo <= prm->hi)) return SIP_ERR_PARAM;
      auto grab = [&](const double* src, std::vector<double>& dst) {
        dst.resize(hs.M);
        if (is_device_ptr(src)) CU(cudaMemcpy(dst.data(), src, hs.M * sizeof(double), cudaMemcpyDeviceToHost));
        else memcpy(dst.data(), src, hs.M * sizeof(double));
      };
      if (prm->lo_vec) grab(prm->lo_vec, hs.lo_vec);
      if (prm->hi_vec) grab(prm->hi_vec, hs.hi_vec);
      for (int64_t q = 0; q < hs.M; ++q) {
        const double lo = hs.lo_vec.empty() ? prm->lo : hs.lo_vec[q];
        const double hi = hs.hi_vec.empty() ? prm->hi : hs.hi_vec[q];
        if (!(lo <= hi)) return SIP_ERR_PARAM;
        if (lo > 0.0 || hi < 0.0) hs.zero_in = 0;
      }
      if (hs.M == 0 && (prm->lo > 0.0 || prm->hi < 0.0)) hs.zero_in = 0;
    } else if (type == SIP_SET_L1_BALL || type == SIP_SET_L2_BALL) {
      if (!(prm->sigma >= 0)) return SIP_ERR_PARAM;
    } else if (type == SIP_SET_ANNULUS) {
      if (!(prm->sigma_lo >= 0) || !(prm->sigma_lo <= prm->sigma_hi)) return SIP_ERR_PARAM;
      hs.zero_in = prm->sigma_lo <= 0.0;
    } else if (type == SIP_SET_CARDINALITY) {
      if (prm->relative) { if (!(prm->k_frac >= 0 && prm->k_frac <= 1)) return SIP_ERR_PARAM; }
      else if (prm->k < 0 || prm->k > hs.M) return SIP_ERR_PARAM;
    } else if (type == SIP_SET_DCT_L1 || type == SIP_SET_HAAR_L1) {   // {x : ||D x||_1 <= sigma}, D orthonormal
      if (type == SIP_SET_HAAR_L1) {
        const long long ax[3] = {nz, ny, nx};
        for (int a = 0; a < 3; ++a)
          if (ax[a] < 1 || (ax[a] & (ax[a] - 1))) { g->err = "Haar l1 sets need every grid axis a power of two"; return SIP_ERR_CONFIG; }
      }
      if (op != SIP_OP_IDENTITY) { g->err = "transform-domain l1 sets keep the transform inside the set: op must be IDENTITY"; return SIP_ERR_CONFIG; }
      if (g->nranks > 1) { g->err = "transform-domain l1 sets: one rank only"; return SIP_ERR_CONFIG; }
      if (!(prm->sigma >= 0)) return SIP_ERR_PARAM;
      if (prm->app_mode != SIP_APPLY_WHOLE) { g->err = "transform-domain l1 sets act on the whole grid"; return SIP_ERR_CONFIG; }
    } else if (type == SIP_SET_RANK || type == SIP_SET_NUCLEAR) {
      // matrix view (reading L29); the batched Jacobi kernel's limits
      if (op == SIP_OP_TV || op == SIP_OP_BLUR_MASK) { g->err = "rank / nuclear sets need a single-block operator"; return SIP_ERR_CONFIG; }
      if (g->nranks > 1) { g->err = "rank / nuclear sets: one rank only"; return SIP_ERR_CONFIG; }
      const int prim = op == SIP_OP_IDENTITY ? PRIM_I : op == SIP_OP_DZ ? PRIM_Z : op == SIP_OP_DY ? PRIM_Y : PRIM_X;
      const MatView mv = mat_view(g->ndim, (int)nz, (int)ny, (int)nx, prim);
      if (mv.n > SVD_NMAX || mv.n < 1) { g->err = "rank / nuclear sets: min(rows, cols) of the matrix view must be 1..2048"; return SIP_ERR_CONFIG; }
      if (type == SIP_SET_RANK && (prm->relative || prm->k < 0)) return SIP_ERR_PARAM;
      if (type == SIP_SET_NUCLEAR && !(prm->sigma >= 0)) return SIP_ERR_PARAM;
      if (prm->app_mode != SIP_APPLY_WHOLE) { g->err = "rank / nuclear sets act on whole matrices"; return SIP_ERR_CONFIG; }
    }
    // per-fiber application (NEXT-1)
    if (prm->app_mode < SIP_APPLY_WHOLE || prm->app_mode > SIP_APPLY_Z_FIBERS) return SIP_ERR_ARG;
    hs.fib = 0;
    hs.flen = 0;
    if (prm->app_mode != SIP_APPLY_WHOLE && type != SIP_SET_BOUNDS) {   // bounds: separable, same set
      if (type != SIP_SET_CARDINALITY && type != SIP_SET_L1_BALL && type != SIP_SET_L2_BALL && type != SIP_SET_ANNULUS) {
        g->err = "per-fiber sets: cardinality, l1 ball, l2 ball, annulus";
        return SIP_ERR_CONFIG;
      }
      if (op == SIP_OP_TV || op == SIP_OP_BLUR_MASK) { g->err = "per-fiber sets need a single-block operator"; return SIP_ERR_CONFIG; }
      if (type != SIP_SET_CARDINALITY && prm->relative) return SIP_ERR_PARAM;   // norm radii per fiber: absolute (L28)
      hs.fib = prm->app_mode;
      hs.flen = prm->app_mode == SIP_APPLY_X_FIBERS ? nx - (op == SIP_OP_DX ? 1 : 0) : nz - (op == SIP_OP_DZ ? 1 : 0);
      if (hs.flen > 4096) { g->err = "per-fiber sets: fibers longer than 4096"; return SIP_ERR_CONFIG; }
      if (type == SIP_SET_CARDINALITY && !prm->relative && prm->k > hs.flen) return SIP_ERR_PARAM;
    }
    g->sets.push_back(std::move(hs));
    g->eng.reset();
    g->levels.clear();
    g->last = nullptr; g->last_team = nullptr;
    if (set_id) *set_id = (int)g->sets.size() - 1;
    return SIP_OK;
  });
}

sip_status sip_set_option(sip_grid g, const char* key, double value) {
  if (!g || !key) return SIP_ERR_ARG;
  std::string k(key);
  Options& o = g->opt;
  if (k == "rho0") { if (!(value > 0)) return SIP_ERR_PARAM; o.rho0 = value; }
  else if (k == "gamma0") { if (!(value >= 1 && value < 2)) return SIP_ERR_PARAM; o.gamma0 = value; }
  else if (k == "n_cg") { if (value < 0) return SIP_ERR_PARAM; o.n_cg = (int)value; }
  else if (k == "eq25") o.eq25 = value != 0;
  else if (k == "fixed_work") o.fixed_work = value != 0;
  else if (k == "eps_evol") o.eps_evol = value;
  else if (k == "eps_corr") o.eps_corr = value;
  else if (k == "adapt_every") { if (value != 2) { g->err = "adapt_every must be 2 (ping-pong snapshots)"; return SIP_ERR_PARAM; } o.adapt_every = 2; }
  else if (k == "check_every") { if (value < 1) return SIP_ERR_PARAM; o.check_every = (int)value; }
  else if (k == "rho_ratio_cap") { if (!(value >= 1)) return SIP_ERR_PARAM; o.rho_ratio_cap = value; }
  else if (k == "gamma_max") { if (!(value >= 1 && value < 2)) return SIP_ERR_PARAM; o.gamma_max = value; }
  else if (k == "cg_tol_floor") o.cg_tol_floor = value;
  else if (k == "warm_start") o.warm_start = value != 0;
  else if (k == "graph_iters") { if (value < 0) return SIP_ERR_PARAM; o.graph_iters = (int)value; }
  else if (k == "profile") o.profile = value != 0;
  else if (k == "virtual_ranks") {
    const int G = (int)value;
    if (G < 1 || (double)G != value || G > g->n[0]) return SIP_ERR_PARAM;
    if (g->nranks > 1) { g->err = "virtual_ranks on an NCCL grid"; return SIP_ERR_CONFIG; }
    if (G != g->vranks) {
      if (g->stream) cudaStreamSynchronize(g->stream);
      g->eng.reset(); g->levels.clear(); g->last = nullptr; g->last_team = nullptr; g->comm.reset();
      g->vranks = G;
    }
  }
  else { g->err = "unknown option " + k; return SIP_ERR_ARG; }
  return SIP_OK;
}

sip_status sip_project(sip_grid g, const void* m, void* x, int max_iter, double tol, sip_result* res) {
  if (!g || !m || !x || max_iter < 1 || m == x) return SIP_ERR_ARG;
  return guarded(g, [&]() -> sip_status {
    return g->dtype == SIP_F32 ? project_T<float>(g, m, x, max_iter, tol, res)
                               : project_T<double>(g, m, x, max_iter, tol, res);
  });
}

sip_status sip_project_multilevel(sip_grid g, const void* m, void* x, int n_levels, int coarsen,
                                  int max_iter, double tol, sip_result* per_level) {
  if (!g || !m || !x || n_levels < 1 || coarsen != 2 || max_iter < 1 || m == x) return SIP_ERR_ARG;
  for (auto& s : g->sets)
    if (s.op == SIP_OP_BLUR_MASK || !s.lo_vec.empty() || !s.hi_vec.empty()) {
      g->err = "multilevel: blur/mask operators and per-entry bounds are not supported";
      return SIP_ERR_CONFIG;
    }
  const int f = 1 << (n_levels - 1);
  for (int a = 0; a < 3; ++a) {
    if (a == 1 && g->ndim == 2) continue;
    if (g->n[a] % f != 0 || g->n[a] / f < 2) { g->err = "grid not divisible for the levels"; return SIP_ERR_CONFIG; }
  }
  return guarded(g, [&]() -> sip_status {
    if (is_team(g))
      return g->dtype == SIP_F32 ? multilevel_team_T<float>(g, m, x, n_levels, max_iter, tol, per_level)
                                 : multilevel_team_T<double>(g, m, x, n_levels, max_iter, tol, per_level);
    return g->dtype == SIP_F32 ? multilevel_T<float>(g, m, x, n_levels, max_iter, tol, per_level)
                               : multilevel_T<double>(g, m, x, n_levels, max_iter, tol, per_level);
  });
}

void sip_destroy(sip_grid g) {
  if (!g) return;
  int cur;
  if (cudaGetDevice(&cur) == cudaSuccess && cur != g->device) cudaSetDevice(g->device);
  if (g->stream) cudaStreamSynchronize(g->stream);
  g->levels.clear();
  g->eng.reset();
  if (g->fence) cudaEventDestroy(g->fence);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

sip_status sip_apply_op(sip_grid g, int set_id, const void* x, void* y) {
  if (!g || !x || !y || set_id < 0 || set_id >= (int)g->sets.size()) return SIP_ERR_ARG;
  return guarded(g, [&]() -> sip_status {
    return g->dtype == SIP_F32 ? apply_op_T<float>(g, set_id, x, y) : apply_op_T<double>(g, set_id, x, y);
  });
}

sip_status sip_apply_system(sip_grid g, const double* rho, const void* p, void* q) {
  if (!g || !rho || !p || !q) return SIP_ERR_ARG;
  return guarded(g, [&]() -> sip_status {
    return g->dtype == SIP_F32 ? apply_system_T<float>(g, rho, p, q) : apply_system_T<double>(g, rho, p, q);
  });
}

sip_status sip_cg(sip_grid g, const double* rho, const void* b, void* x, int n_cg, int eq25, int* iterations) {
  if (!g || !rho || !b || !x || n_cg < 0) return SIP_ERR_ARG;
  return guarded(g, [&]() -> sip_status {
    return g->dtype == SIP_F32 ? cg_T<float>(g, rho, b, x, n_cg, eq25, iterations)
                               : cg_T<double>(g, rho, b, x, n_cg, eq25, iterations);
  });
}

sip_status sip_project_set(sip_grid g, int set_id, const void* w, void* y) {
  if (!g || !w || !y || set_id < 0 || set_id >= (int)g->sets.size()) return SIP_ERR_ARG;
  return guarded(g, [&]() -> sip_status {
    return g->dtype == SIP_F32 ? project_set_T<float>(g, set_id, w, y) : project_set_T<double>(g, set_id, w, y);
  });
}

sip_status sip_get_state(sip_grid g, int set_id, int which, void* out) {
  if (!g || !out || set_id < 0 || set_id > (int)g->sets.size() || (which != 0 && which != 1)) return SIP_ERR_ARG;
  return guarded(g, [&]() -> sip_status {
    if (is_team(g))
      return g->dtype == SIP_F32 ? get_state_team_T<float>(g, set_id, which, out)
                                 : get_state_team_T<double>(g, set_id, which, out);
    return g->dtype == SIP_F32 ? get_state_T<float>(g, set_id, which, out) : get_state_T<double>(g, set_id, which, out);
  });
}

sip_status sip_get_log(sip_grid g, int max_iter, int* cg, int* branch, double* rho_trace,
                       double* gamma_trace, double* r_feas, double* r_evol) {
  if (!g || max_iter < 0) return SIP_ERR_ARG;
  return guarded(g, [&]() -> sip_status {
    return g->dtype == SIP_F32 ? get_log_T<float>(g, max_iter, cg, branch, rho_trace, gamma_trace, r_feas, r_evol)
                               : get_log_T<double>(g, max_iter, cg, branch, rho_trace, gamma_trace, r_feas, r_evol);
  });
}

sip_status sip_get_support_log(sip_grid g, int max_iter, uint64_t* out) {
  if (!g || !out || max_iter < 0) return SIP_ERR_ARG;
  return guarded(g, [&]() -> sip_status {
    auto run = [&](auto tag) -> sip_status {
      using T = decltype(tag);
      std::vector<Engine<T>*> es;
      if (is_team(g) && g->last_team) {
        for (auto& e : static_cast<Team<T>*>(g->last_team)->eng) es.push_back(e.get());
      } else {
        es.push_back(last_engine<T>(g));
      }
      const int p = es[0]->p;
      memset(out, 0, (size_t)max_iter * std::max(p, 0) * sizeof(uint64_t));
      std::vector<uint64_t> tmp;
      for (Engine<T>* e : es) {
        if (!e->ran) throw SipError{SIP_ERR_STATE, "no projection log"};
        const int n = std::min(max_iter, e->log_cap);
        tmp.assign((size_t)n * std::max(p, 1), 0);
        if (p) CU(cudaMemcpy(tmp.data(), e->d_log_supp, (size_t)n * p * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        for (size_t q = 0; q < (size_t)n * p; ++q) out[q] += tmp[q];
      }
      return SIP_OK;
    };
    return g->dtype == SIP_F32 ? run(float()) : run(double());
  });
}

sip_status sip_dykstra(sip_grid g, const void* m, void* x, int max_outer, double tol, int inner_max_iter,
                       double inner_tol, sip_dykstra_log* log) {
  if (!g || !m || !x || max_outer < 1 || inner_max_iter < 1) return SIP_ERR_ARG;
  return guarded(g, [&]() -> sip_status {
    return g->dtype == SIP_F32 ? dykstra_T<float>(g, m, x, max_outer, tol, inner_max_iter, inner_tol, log)
                               : dykstra_T<double>(g, m, x, max_outer, tol, inner_max_iter, inner_tol, log);
  });
}

sip_status sip_get_sizes(sip_grid g, int* p, int64_t* n_local, int set_id, int64_t* m_compact) {
  if (!g) return SIP_ERR_ARG;
  if (p) *p = (int)g->sets.size();
  if (n_local) {
    int z0 = 0, nzl = (int)g->n[0];
    if (g->nranks > 1) slab_of((int)g->n[0], g->nranks, g->rank, &z0, &nzl);
    *n_local = (int64_t)nzl * g->n[1] * g->n[2];
  }
  if (m_compact) {
    if (set_id < 0 || set_id > (int)g->sets.size()) return SIP_ERR_ARG;
    *m_compact = set_id == (int)g->sets.size() ? g->n[0] * g->n[1] * g->n[2] : g->sets[set_id].M;
  }
  return SIP_OK;
}

sip_status sip_get_profile(sip_grid g, int n, double* ms, int64_t* count) {
  if (!g || n < 0) return SIP_ERR_ARG;
  return guarded(g, [&]() -> sip_status {
    if (!g->last) throw SipError{SIP_ERR_STATE, "no projection"};
    auto fill = [&](auto* e) {
      for (int q = 0; q < n && q < Engine<float>::NKIND; ++q) {
        if (ms) ms[q] = e->prof_ms[q];
        if (count) count[q] = e->prof_cnt[q];
      }
    };
    if (g->dtype == SIP_F32) fill(static_cast<Engine<float>*>(g->last));
    else fill(static_cast<Engine<double>*>(g->last));
    return SIP_OK;
  });
}

sip_status sip_get_launch_count(sip_grid g, int64_t* launches) {
  if (!g || !launches) return SIP_ERR_ARG;
  *launches = g->last_launches;
  return SIP_OK;
}

}  // extern "C"
