// wq_dev.cuh -- device helpers of the row-block kernels: compile-time
// dispatch of staircase offsets, unrolling, shared-memory addressing, TMA
// bulk / tensor copies and mbarrier primitives (sm_100a PTX).
#pragma once
#include <type_traits>
#include <stdint.h>

namespace wqdev {

// compile-time dispatch of a runtime offset o in [LO, HI] (|o| <= 31): f(integral_constant<o>);
// a dense switch, compiled to a jump table (one indirect branch, uniform across the warp)
#define WQ_CASE(O) \
    case O:        \
        if constexpr ((O) >= LO && (O) <= HI) f(std::integral_constant<int, (O)>{}); \
        break;
#define WQ_CASE8(B) WQ_CASE(B) WQ_CASE(B + 1) WQ_CASE(B + 2) WQ_CASE(B + 3) WQ_CASE(B + 4) WQ_CASE(B + 5) WQ_CASE(B + 6) WQ_CASE(B + 7)
template <int LO, int HI, class F>
__device__ __forceinline__ void dispatch(int o, F &&f) {
    static_assert(LO >= -32 && HI < 32, "dispatch range");
    switch (o) {
        WQ_CASE8(-32) WQ_CASE8(-24) WQ_CASE8(-16) WQ_CASE8(-8) WQ_CASE8(0) WQ_CASE8(8) WQ_CASE8(16) WQ_CASE8(24)
    default: break;
    }
}
#undef WQ_CASE8
#undef WQ_CASE

template <int N, class F>
__device__ __forceinline__ void unroll(F &&f) {
    if constexpr (N > 0) {
        unroll<N - 1>(f);
        f(std::integral_constant<int, N - 1>{});
    }
}

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(b)) : "memory");
}
// relaxed arrive: no release ordering of this thread's earlier memory operations (used by
// consumers to hand a ring slot back once the values read from it have been consumed by
// arithmetic; a release arrive would also wait for the warp's outstanding global stores)
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t *b) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.relaxed.cta.shared::cta.b64 st, [%0];\n}" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, unsigned bytes) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
// try_wait with a suspend-time hint: the waiting warp sleeps in hardware (up to ~0.1 ms) until the
// phase completes instead of re-issuing the test
#ifndef WQ_MBAR_HINT
#define WQ_MBAR_HINT 100000
#endif
__device__ __forceinline__ bool mbar_try(uint64_t *b, unsigned parity) {
    unsigned ok;
#if WQ_MBAR_HINT > 0
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity), "r"((unsigned)WQ_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
#endif
    return ok != 0;
}
// wait until the phase with the given parity has completed
// (fails loudly with a trap instead of hanging if a pipeline invariant is ever broken)
#ifdef WQ_DIAG
// debug builds: on a stuck wait, record (block, thread, barrier offset, parity) in host-mapped memory
static __device__ unsigned long long *g_wq_diag;
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
    unsigned spins = 0;
    while (!mbar_try(b, parity)) {
#ifdef WQ_DIAG
        if (++spins > (1u << 22)) {
            if (g_wq_diag) {
                unsigned long long k = atomicAdd(&g_wq_diag[0], 1ull);
                if (k < 64) {
                    volatile unsigned long long *d = g_wq_diag + 1 + 2 * k;
                    d[0] = ((unsigned long long)blockIdx.x << 32) | threadIdx.x;
                    d[1] = ((unsigned long long)smem_u32(b) << 32) | parity;
                    __threadfence_system();
                }
            }
            asm volatile("exit;");
        }
#else
        if (++spins > (1u << 26)) __trap();
#endif
    }
}

// wait with a nanosleep back-off after each failed test: for roles that wait long (a whole pipeline
// step), so that their re-tests do not take issue slots from the warps doing the work
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *b, unsigned parity) {
    unsigned spins = 0;
    while (!mbar_try(b, parity)) {
        __nanosleep(256);
        if (++spins > (1u << 25)) __trap();
    }
}

// 16-B asynchronous global -> shared copy (L2 only); src_bytes < 16 zero-fills the rest
__device__ __forceinline__ void cp_async16(void *dst, const void *src, unsigned src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------- named barrier (subset of warps)
__device__ __forceinline__ void bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- TMA
// shared -> global bulk copy (async proxy); addresses 16-B aligned, bytes % 16 == 0
__device__ __forceinline__ void bulk_s2g(void *g, const void *s, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// generic-proxy shared writes -> visible to the async proxy (before a bulk copy reads them)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 4D tensor tile global -> shared, completion counted on an mbarrier (bytes)
__device__ __forceinline__ void tma_load_4d(void *dst, const void *tmap, uint64_t *bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

}  // namespace wqdev
