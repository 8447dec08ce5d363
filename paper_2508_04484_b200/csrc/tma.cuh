// Bulk-copy TMA (cp.async.bulk) + mbarrier helpers for the streaming kernels.
//
// Every n-side matrix is cell-major with zero halo rows around it (pnd.h), so
// the rows a chunk needs -- stencil reach included -- are contiguous, in-bounds
// byte ranges: one cp.async.bulk each, completing on an mbarrier. No tensor
// map is needed for this layout (the column-blocked layout of ranks above 64
// keeps every block contiguous the same way, csrc/xwide.cu).
#pragma once

#include "pnd.h"

namespace pnd {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

#ifndef PND_MBAR_SPIN
#define PND_MBAR_SPIN 1
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
#if PND_MBAR_SPIN
  // spin on test_wait: a suspended try_wait wakes late, and these waits sit
  // on the per-chunk critical path of the producer/former/contraction chain
  unsigned ok;
  do {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}

// mbarrier wait for a thread that is normally early (the producer): back off
// with nanosleep instead of spinning on the issue slots the workers need
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, unsigned parity) {
  while (!mbar_test(bar, parity)) __nanosleep(200);
}

// arrive (count 1) on an mbarrier; release semantics order this thread's prior writes
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// named barrier over a subset of the CTA's warps
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

}  // namespace pnd

namespace pnd {

// one contiguous global -> shared copy through the TMA engine (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"((unsigned long long)src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// prefetch a contiguous global range into L2 (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"((unsigned long long)src),
               "r"(bytes)
               : "memory");
}

// ring position of iteration it: slot s, use count k (phase parity k & 1)
struct Ring {
  int s = 0, k = 0, n;
  __device__ explicit Ring(int n_) : n(n_) {}
  __device__ void next() {
    if (++s == n) {
      s = 0;
      ++k;
    }
  }
};

// one elected lane signals for the whole warp
__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
}

}  // namespace pnd
