// pff_bulk.cuh -- TMA bulk copies (cp.async.bulk) and mbarrier helpers shared
// by the write-once sweep kernels (pff_sweep.cu: Q2, pff_sweep4.cu: Q4).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// PFF_DEBUG_CHECKS (debug build, tools/debug_checks.sh): device-side bounds and
// protocol checks of the TMA / mbarrier staging -- compute-sanitizer is not
// available on the GPU pool, so the staging rings assert their own invariants
#ifdef PFF_DEBUG_CHECKS
#include <cstdio>
#define PFF_DCHECK(cond)                                                                   \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("PFF_DCHECK failed %s:%d: %s (block %d lane %d)\n", __FILE__, __LINE__,  \
                   #cond, (int)blockIdx.x, (int)threadIdx.x);                              \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define PFF_DCHECK(cond) do { } while (0)
#endif

namespace pff {
namespace bulk {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)),
                 "r"(bytes) : "memory");
}
#ifdef PFF_DEBUG_CHECKS
// bounded wait: a parity that never completes (lost or mis-sized copy) traps
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    for (long long it = 0;; ++it) {
        unsigned done;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(smem_u32(b)), "r"(parity) : "memory");
        if (done) return;
        PFF_DCHECK(it < (1ll << 26));
    }
}
#else
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
#endif
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* b) {
    PFF_DCHECK((smem_u32(dst) & 15u) == 0 && (((uintptr_t)src) & 15u) == 0 && (bytes & 15u) == 0 &&
               bytes > 0);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}


}  // namespace bulk
}  // namespace pff
