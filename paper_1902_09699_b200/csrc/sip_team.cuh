// sip_team.cuh -- the finalisers of the z-slab decomposition.
//
// On one rank every reducing kernel ends with its last CTA taking the
// decision (alpha, beta, the Eq. 25 flags, the radix digit, ...).  On a
// z-slab of nranks > 1 the last CTA instead publishes the rank-local values
// to its slot of the gather buffer (Prob::xg); the runtime exchanges the
// slots (NCCL send/recv over NVLink, or device copies between the slabs of
// one device) together with the 1-plane halos, and k_fin sums the slots in
// rank order 0..G-1 -- the same bits on every rank -- and runs the same
// finaliser as the single-rank path.  Integer histograms (radix select) and
// tie counts are exact; fp64 sums differ from the one-rank order only by
// rounding.
#pragma once
#include "sip_pass.cuh"

namespace sip {

enum Site { ST_INIT = 0, ST_RHS = 1, ST_CG1 = 2, ST_CG2 = 3, ST_PASS1 = 4, ST_SELECT = 5, ST_TIE = 6,
            ST_PASS2 = 7 };

constexpr int FIN_MAXV = MAXP * NSLOT + NEVOL;   // largest double payload (pass 1)

// gather payload (doubles) of a site
__host__ inline int site_payload(int site, int P, int njobs) {
  switch (site) {
    case ST_INIT: return 2 * P;
    case ST_RHS: return 2;
    case ST_CG1: case ST_CG2: return 1;
    case ST_PASS1: return P * NSLOT + NEVOL;
    case ST_SELECT: return njobs * HJOB;
    case ST_TIE: return 3 * P;
    default: return 4 * P;
  }
}

// radix round `round` of every active job on the summed histograms
template <class T>
__device__ inline void fin_select(const Prob<T>& P, Ctrl& C, int round) {
  const bool check = (C.k % C.opt.check_every) == 0;
  for (int jb = 0; jb < C.njobs; ++jb) {
    Job& J = C.job[jb];
    if (J.mode != JM_SEARCH || J.round != round - 1 || (J.on_s && !check)) continue;
    unsigned* gc = P.gh_cnt + (size_t)jb * NBUCK;
    unsigned long long* g0 = P.gh_s0 + (size_t)jb * NBUCK;
    unsigned long long* g1 = P.gh_s1 + (size_t)jb * NBUCK;
    for (int d = threadIdx.x; d < NBUCK; d += BLOCK) {
      unsigned long long a0 = 0, a1 = 0;
      unsigned c = 0;
      for (int r = 0; r < P.nranks; ++r) {
        const unsigned long long* s0 =
            reinterpret_cast<const unsigned long long*>(P.xg + (size_t)r * P.xslot + (size_t)jb * HJOB);
        const unsigned long long* s1 = s0 + NBUCK;
        const unsigned* cn = reinterpret_cast<const unsigned*>(s1 + NBUCK);
        a0 += s0[d]; a1 += s1[d]; c += cn[d];
      }
      g0[d] = a0; g1[d] = a1; gc[d] = c;
    }
    __syncthreads();
    resolve_round<T>(P, J, round, gc, g0, g1);
    __syncthreads();
    for (int d = threadIdx.x; d < NBUCK; d += BLOCK) { gc[d] = 0u; g0[d] = 0ull; g1[d] = 0ull; }
    __syncthreads();
  }
}

// cardinality ties: global index order is block-major, then rank, then the
// local order, so the offset of this rank's tiles of block bl is the ties of
// every rank in blocks < bl plus those of lower ranks in block bl (L6)
template <class T>
__device__ inline void fin_tie(const Prob<T>& P, Ctrl& C) {
  constexpr int W = VT<T>::W;
  __shared__ long long add[3];
  const int nch = P.g.N / W;
  const int tpb = (nch + BLOCK - 1) / BLOCK;
  for (int i = 0; i < P.P; ++i) {
    const SetD<T>& S = P.set[i];
    if (S.kind != K_CARD || S.job < 0) continue;
    const Job& J = C.job[S.job];
    if (J.mode != JM_DONE || !J.ties) continue;
    if (threadIdx.x == 0) {
      long long before_all = 0, mine_before = 0;
      for (int bl = 0; bl < S.nblk; ++bl) {
        long long lower = 0, all = 0;
        for (int r = 0; r < P.nranks; ++r) {
          const long long c = (long long)P.xg[(size_t)r * P.xslot + i * 3 + bl];
          if (r < P.rank) lower += c;
          all += c;
        }
        add[bl] = before_all + lower - mine_before;   // the local scan already counts my blocks < bl
        before_all += all;
        mine_before += (long long)P.xg[(size_t)P.rank * P.xslot + i * 3 + bl];
      }
    }
    __syncthreads();
    int* tc = P.tiecnt + (size_t)S.job * P.ntiles_max;
    for (int bl = 0; bl < S.nblk; ++bl)
      for (int t = bl * tpb + threadIdx.x; t < (bl + 1) * tpb; t += BLOCK) tc[t] += (int)add[bl];
    __syncthreads();
  }
}

// one CTA: sum the gathered slots in rank order, then the site's finaliser.
// The early exits mirror those of the kernel that published (same Ctrl).
template <class T>
__global__ void __launch_bounds__(BLOCK) k_fin(const __grid_constant__ Prob<T> P, int site, int j, int round) {
  Ctrl& C = *P.ctrl;
  __shared__ double v[FIN_MAXV];
  auto gsum = [&](int n) {
    for (int i = threadIdx.x; i < n; i += BLOCK) {
      double a = 0.0;
      for (int r = 0; r < P.nranks; ++r) a += P.xg[(size_t)r * P.xslot + i];
      v[i] = a;
    }
    __syncthreads();
  };
  switch (site) {
    case ST_INIT:
      gsum(2 * P.P);
      if (threadIdx.x == 0) fin_init<T>(P, C, v);
      break;
    case ST_RHS:
      if (C.stopped) return;
      gsum(2);
      if (threadIdx.x == 0) fin_rhs(C, v);
      break;
    case ST_CG1:
      if (C.stopped || (j == 0 && C.zero_x) || !C.cg_active) return;
      gsum(1);
      if (threadIdx.x == 0) fin_cg1(C, v, j);
      break;
    case ST_CG2:
      if (C.stopped || !C.cg_active) return;
      gsum(1);
      if (threadIdx.x == 0) fin_cg2(C, v, j);
      break;
    case ST_PASS1:
      if (C.stopped) return;
      gsum(P.P * NSLOT + NEVOL);
      fin_pass1<T>(P, C, v);
      break;
    case ST_SELECT:
      if (C.stopped) return;
      fin_select<T>(P, C, round);
      break;
    case ST_TIE:
      if (C.stopped) return;
      fin_tie<T>(P, C);
      break;
    default:
      if (C.stopped) return;
      gsum(4 * P.P);
      fin_pass2<T>(P, C, v);
  }
}

}  // namespace sip
