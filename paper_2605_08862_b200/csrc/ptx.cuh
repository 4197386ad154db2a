// ptx.cuh — thin inline-PTX wrappers for sm_100a: mbarrier, 1-D bulk copy (TMA), cache hints.
#pragma once
#include <cstdint>
#include <cstdio>

namespace bs {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// try_wait with a suspend-time hint: a waiting warp sleeps (NANOSLEEP.SYNCS) until the phase
// completes or the hint expires instead of spinning, so waiting warps do not take issue
// slots from the working ones.
constexpr uint32_t MBAR_SUSPEND_NS = 1000000u;

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase), "r"(MBAR_SUSPEND_NS)
        : "memory");
    return ok != 0;
}

// Cluster-scope wait: relaxed polls, one acquire fence once the phase has completed.
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase), "r"(MBAR_SUSPEND_NS)
        : "memory");
    if (ok) asm volatile("fence.acquire.cluster;" ::: "memory");
    return ok != 0;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Watchdog: a wait that has not completed after ~4 s is a protocol bug; trap (the launch
// fails with an error) instead of hanging the device.
__device__ __noinline__ void mbar_wait_slow(uint64_t* bar, uint32_t phase, bool cluster) {
    const uint64_t t0 = globaltimer_ns();
    for (uint32_t it = 1;; ++it) {
        if (cluster ? mbar_try_wait_cluster(bar, phase) : mbar_try_wait(bar, phase)) return;
        if ((it & 15u) == 0 && globaltimer_ns() - t0 > 3000000000ull) {
#ifdef BS_TRACE
            printf("bs watchdog: block %d thread %d mbarrier smem+0x%x phase %u\n", (int)blockIdx.x,
                   (int)threadIdx.x, smem_u32(bar), phase);
#endif
            __trap();
        }
    }
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    if (!mbar_try_wait(bar, phase)) mbar_wait_slow(bar, phase, false);
}

// Wait with acquire at CLUSTER scope (for barriers that peers arrive on remotely).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
    if (!mbar_try_wait_cluster(bar, phase)) mbar_wait_slow(bar, phase, true);
}

// Arrive (release, cluster scope) on the mbarrier at the same smem offset in CTA `rank`.
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
    asm volatile(
        "{\n"
        ".reg .b32 ra;\n"
        "mapa.shared::cluster.u32 ra, %0, %1;\n"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(rank)
        : "memory");
}

// 16-byte asynchronous store into CTA `rank`'s shared memory at the offset of `dst`,
// completing 16 transaction bytes on that CTA's mbarrier at the offset of `bar`
// (st.async: no fence, the data and the completion signal travel together).
__device__ __forceinline__ void st_async_v4(void* dst, uint4 v, uint64_t* bar, uint32_t rank) {
    asm volatile(
        "{\n"
        ".reg .b32 ra, rb;\n"
        "mapa.shared::cluster.u32 ra, %0, %6;\n"
        "mapa.shared::cluster.u32 rb, %1, %6;\n"
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [ra], {%2, %3, %4, %5}, [rb];\n"
        "}\n" ::"r"(smem_u32(dst)),
        "r"(smem_u32(bar)), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rank)
        : "memory");
}

// L2 eviction-first policy for streamed logits (keeps the draft index resident in L2).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// 1-D bulk async copy global -> shared (TMA engine), completion on an mbarrier.
// dst, src 16-B aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// GPU-scope acquire / release / relaxed global accesses (the verify scheduler's queues).
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)));
    return v;
}

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
    uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    lo = __shfl_xor_sync(0xFFFFFFFFu, lo, m);
    hi = __shfl_xor_sync(0xFFFFFFFFu, hi, m);
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t shfl_up_u64(uint64_t v, int d) {
    uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    lo = __shfl_up_sync(0xFFFFFFFFu, lo, d);
    hi = __shfl_up_sync(0xFFFFFFFFu, hi, d);
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
    uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    lo = __shfl_sync(0xFFFFFFFFu, lo, src);
    hi = __shfl_sync(0xFFFFFFFFu, hi, src);
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int m = 16; m; m >>= 1) v += shfl_xor_u64(v, m);
    return v;
}

__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        uint64_t o = shfl_up_u64(v, d);
        if (lane >= d) v += o;
    }
    return v;
}

}  // namespace bs
