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

// A two-stage ring of up to NA arrays of one tile each (tile = `tile`
// chunks of 16 bytes, plus one spare chunk per array for an x neighbour).
// All threads of the CTA construct it identically; thread 0 issues.
template <int NA>
struct Stage2 {
  uint64_t* bar;      // [2] mbarriers (shared)
  char* buf;          // [2][NA][slot] (shared, 16-byte aligned)
  int slot;           // bytes per array slot = (tile + 1) * 16
  unsigned phase;     // bit s: parity of stage s's next completion

  __device__ void init(uint64_t* bars, char* b, int tile) {
    bar = bars;
    buf = b;
    slot = (tile + 1) * 16;
    phase = 0;
    if (threadIdx.x == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      mbar_fence_init();
    }
    __syncthreads();
  }
  __device__ __forceinline__ char* at(int s, int a) const { return buf + ((size_t)s * NA + a) * slot; }
  // thread 0: copy bytes[a] from src[a] into stage s, array a (na arrays)
  __device__ __forceinline__ void issue(int s, int na, const char* const* src, const unsigned* bytes) {
    if (threadIdx.x == 0) {
      unsigned tot = 0;
      for (int a = 0; a < na; ++a) tot += bytes[a];
      mbar_expect_tx(&bar[s], tot);
      for (int a = 0; a < na; ++a)
        if (bytes[a]) bulk_g2s(at(s, a), src[a], bytes[a], &bar[s]);
    }
  }
  __device__ __forceinline__ void wait(int s) {
    mbar_wait(&bar[s], (phase >> s) & 1u);
    phase ^= 1u << s;
  }
};

}  // namespace sip
