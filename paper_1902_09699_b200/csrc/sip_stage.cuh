// sip_stage.cuh -- double-buffered 1D bulk-copy staging (sm_90+/sm_100a).
//
// The streaming kernels read several arrays over the same contiguous chunk
// range.  Instead of holding every load in flight in registers, one thread
// issues cp.async.bulk copies (SASS UBLKCP) of the next tile of each array
// into shared memory, armed on an mbarrier with the byte count
// (mbarrier.arrive.expect_tx); the CTA computes the current tile from shared
// memory meanwhile.  Memory-level parallelism then comes from the bulk
// copies (up to one full tile per array per CTA in flight), not from
// occupancy, so register-heavy kernels (Algorithm 2's adapt iterations)
// still stream at HBM rate.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sip {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// the same copy with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// A ring of stages of up to NA arrays of one tile each (tile = `tile`
// chunks of 16 bytes, plus one spare chunk per array for an x neighbour),
// carved from a pool of `pool` array slots: set_layout(mask) packs the
// arrays a consumer uses (bits of mask) into consecutive slots and takes as
// many stages (2..SMAX) as the pool holds, so segments that read few arrays
// keep more tiles in flight.  All threads of the CTA construct it
// identically; thread 0 issues.  A consumer keeps ns - 1 tiles in flight: it
// issues tile t + ns - 1 before it waits for tile t (stage t % ns).  The
// layout may change only when no copy is in flight.
constexpr int SMAX = 8;
template <int NA>
struct Stage2 {
  uint64_t* bar;      // [SMAX] mbarriers (shared)
  char* buf;          // the pool (shared, 16-byte aligned)
  int slot;           // bytes per array slot = (tile + 1) * 16
  int pool;           // array slots in the pool
  int ns;             // stages of the current layout
  int u;              // arrays per stage of the current layout
  unsigned mask;      // arrays of the current layout
  unsigned phase;     // bit s: parity of stage s's next completion

  __device__ void init(uint64_t* bars, char* b, int tile, int pool_slots) {
    bar = bars;
    buf = b;
    slot = (tile + 1) * 16;
    pool = pool_slots;
    phase = 0;
    set_layout((1u << NA) - 1u);
    if (threadIdx.x == 0) {
      for (int q = 0; q < SMAX; ++q) mbar_init(&bar[q], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  __device__ __forceinline__ void set_layout(unsigned m) {
    mask = m;
    u = max(1, __popc(m));
    ns = min(SMAX, max(2, pool / u));
  }
  __device__ __forceinline__ char* at(int s, int a) const {
    return buf + ((size_t)s * u + __popc(mask & ((1u << a) - 1u))) * slot;
  }
  // thread 0: copy bytes[a] from src[a] into stage s, array a (na arrays);
  // hint != 0: arrays in `keep` (bit a) with L2 evict_last, the others with
  // evict_first (hint 2) or the default policy (hint 1)
  __device__ __forceinline__ void issue(int s, int na, const char* const* src, const unsigned* bytes,
                                        int hint = 0, unsigned keep = 0u) {
    if (threadIdx.x == 0) {
      unsigned tot = 0;
      for (int a = 0; a < na; ++a) tot += bytes[a];
      mbar_expect_tx(&bar[s], tot);
      if (hint == 0) {
        for (int a = 0; a < na; ++a)
          if (bytes[a]) bulk_g2s(at(s, a), src[a], bytes[a], &bar[s]);
      } else {
        const uint64_t pl = pol_evict_last(), pf = pol_evict_first();
        for (int a = 0; a < na; ++a) {
          if (!bytes[a]) continue;
          if (keep & (1u << a)) bulk_g2s_hint(at(s, a), src[a], bytes[a], &bar[s], pl);
          else if (hint == 2) bulk_g2s_hint(at(s, a), src[a], bytes[a], &bar[s], pf);
          else bulk_g2s(at(s, a), src[a], bytes[a], &bar[s]);
        }
      }
    }
  }
  __device__ __forceinline__ void wait(int s) {
    mbar_wait(&bar[s], (phase >> s) & 1u);
    phase ^= 1u << s;
  }
};

}  // namespace sip
