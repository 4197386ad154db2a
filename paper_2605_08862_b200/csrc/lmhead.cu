// lmhead.cu — the LM-head GEMM with the verify's first pass fused into its epilogue (SURVEY
// §8(f)3).  logits[r, v] = bf16(sum_k h[r, k] W[v, k]) on the 5th-gen tensor cores, and, while the
// accumulator tile is in registers, the row statistics the verify's max pass computes (readings
// R0/R1: the row maximum of the bf16 logits, the lowest index attaining it, and whether a NaN /
// +inf occurs), folded across the N tiles with one 64-bit atomicMax per (row, tile).  A verify
// launch given those statistics (bsx_set_row_stats) skips its max pass: every CTA of a row's
// cluster publishes the row's precomputed maximum.  (An exact verify cannot also skip the logits
// round trip: its integer masses need the row maximum before any mass.)
//
// Two kernels, the same roles (warp 0 TMA producer, warp 1 MMA issuer, warps 2-5 epilogue over
// the four TMEM lane quarters, two TMEM accumulators so a tile's epilogue overlaps the next
// tile's MMAs, 128-byte-swizzled K-blocks of 64):
//  * lm_head_pair_kernel (default): CTA pairs, tcgen05.mma.cta_group::2 M 256 N 256 K 16, each
//    CTA staging half of the A rows and half of the W rows (32 KB per K-block and SM), 6 stages;
//  * lm_head_kernel (BS_LM_KERNEL=1, kept for measurement): one CTA per SM, M 128 N 256, 48 KB
//    per K-block, 4 stages.
// The epilogue takes each 32-column chunk's maximum with packed bf16 max and falls back to the
// per-element order keys only where R1's ties need it (a chunk straddling V, a NaN / +inf, a
// maximum of +-0).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "../../include/bubblespec.h"
#include "common.cuh"

namespace bs {

#ifndef BS_LM_BN
#define BS_LM_BN 256
#endif
#ifndef BS_LM_ST
#define BS_LM_ST 4
#endif
constexpr int LM_BM = 128, LM_BN = BS_LM_BN, LM_BK = 64, LM_ST = BS_LM_ST, LM_NT = 192;
constexpr uint32_t LM_ABYTES = LM_BM * LM_BK * 2;  // 16 KB
constexpr uint32_t LM_BBYTES = LM_BN * LM_BK * 2;  // 32 KB at N = 256
constexpr size_t LM_SMEM = 1024 + (size_t)LM_ST * (LM_ABYTES + LM_BBYTES) + 256;

struct LmArgs {
    int rows, d, V;
    uint16_t* logits;
    int64_t ld;                 // logits row stride (elements)
    unsigned long long* row_key;  // [rows] (order key of the max << 32) | (~argmax), atomicMax
    uint32_t* row_bad;          // [rows] NaN / +inf seen
};

__device__ __forceinline__ uint32_t lm_s(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void lm_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(lm_s(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void lm_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(lm_s(b)) : "memory");
}
__device__ __forceinline__ void lm_arrive_tx(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lm_s(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void lm_wait(uint64_t* b, uint32_t ph) {
    uint32_t ok = 0;
    uint64_t t0 = 0;
    for (int spin = 0; !ok; ++spin) {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
                     "selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(lm_s(b)), "r"(ph), "r"(1000000u) : "memory");
        if (spin == 64) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        if (spin > 64 && (spin & 255) == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 2000000000ull) __trap();  // 2 s: protocol bug
        }
    }
}
__device__ __forceinline__ void lm_tma(void* dst, const CUtensorMap* m, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(lm_s(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(lm_s(bar)) : "memory");
}
__device__ __forceinline__ uint64_t lm_desc(uint32_t saddr) {  // K-major, 128-byte swizzle
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void lm_ld32(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// packed bf16x2 maximum, NaN-propagating (HMNMX2.NAN)
__device__ __forceinline__ uint32_t lm_hmax2_nan(uint32_t a, uint32_t b) {
    __nv_bfloat162 x, y;
    memcpy(&x, &a, 4);
    memcpy(&y, &b, 4);
    const __nv_bfloat162 z = __hmax2_nan(x, y);
    uint32_t r;
    memcpy(&r, &z, 4);
    return r;
}
// bf16 bits -> 16-bit key ordered like the values (NaN excluded by the caller)
__device__ __forceinline__ uint32_t lm_key(uint32_t b) { return (b & 0x8000u) ? (~b & 0xFFFFu) : (b | 0x8000u); }

// Epilogue of one 128-row x LM_BN-column accumulator (this warp: TMEM lanes q*32.. = rows
// row - lane ..): tcgen05.ld -> bf16 (round to nearest even) -> global stores, and the tile's
// row statistics (best = order key << 16 | ~column, 0 = none; bad = NaN / +inf seen).
__device__ __forceinline__ void lm_drain(const LmArgs& a, uint32_t taddr, int row, int nt, uint32_t& best,
                                         uint32_t& bad) {
    const bool rok = row < a.rows;
    best = 0;
    bad = 0;
    uint16_t* dst = a.logits + (int64_t)(rok ? row : 0) * a.ld + (int64_t)nt * LM_BN;
#pragma unroll 1
    for (int c = 0; c < LM_BN / 32; ++c) {
        uint32_t r[32];
        lm_ld32(taddr + c * 32, r);
        const int col0 = nt * LM_BN + c * 32;
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const __nv_bfloat162 p2 = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
            pk[j] = *reinterpret_cast<const uint32_t*>(&p2);
        }
        // the chunk's maximum with packed NaN-propagating bf16 max (15 HMNMX2); the per-element
        // path only for a chunk that straddles V, holds a NaN / +inf or has a maximum of +-0 (so
        // that the order-key ties of R1 are taken exactly as element by element)
        uint32_t m2 = pk[0];
#pragma unroll
        for (int j = 1; j < 16; ++j) m2 = lm_hmax2_nan(m2, pk[j]);
        const uint32_t mx = lm_hmax2_nan(m2, m2 >> 16) & 0xFFFFu;
        if (col0 + 32 <= a.V && (mx & 0x7FFFu) < 0x7F80u && (mx & 0x7FFFu) != 0u) {
            const uint32_t key = lm_key(mx);
            if (key > (best >> 16)) {  // the first column holding mx (bit-equal: mx is not +-0)
                uint32_t hit = 0;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    hit |= (((pk[j] & 0xFFFFu) == mx) ? 1u : 0u) << (2 * j) | (((pk[j] >> 16) == mx) ? 2u : 0u) << (2 * j);
                best = (key << 16) | (0xFFFFu - (uint32_t)(c * 32 + __ffs(hit) - 1));
            }
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const uint32_t b = (j & 1) ? (pk[j >> 1] >> 16) : (pk[j >> 1] & 0xFFFFu);
                if (col0 + j < a.V) {
                    if ((b & 0x7FFFu) >= 0x7F80u && b != 0xFF80u) {  // NaN or +inf (R0)
                        bad = 1u;
                        if ((b & 0x7FFFu) > 0x7F80u) continue;  // NaN: not a maximum
                    }
                    const uint32_t kv = (lm_key(b) << 16) | (0xFFFFu - (uint32_t)(c * 32 + j));
                    best = max(best, kv);
                }
            }
        }
        if (rok) {
            if (col0 + 32 <= a.V && (((uintptr_t)(dst + c * 32) & 15u) == 0)) {
                uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
                for (int j = 0; j < 4; ++j) d4[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)  // (unrolled: pk stays in registers)
                    if (col0 + j < a.V) dst[c * 32 + j] = (uint16_t)((j & 1) ? (pk[j >> 1] >> 16) : (pk[j >> 1] & 0xFFFFu));
            }
        }
    }
}

// Fold one tile's row statistics into the row's (one 64-bit atomicMax, one atomicOr).
__device__ __forceinline__ void lm_stats(const LmArgs& a, int row, int nt, uint32_t best, uint32_t bad) {
    if (row >= a.rows) return;
    if (best) {
        const uint32_t key = best >> 16, col = (uint32_t)nt * LM_BN + (0xFFFFu - (best & 0xFFFFu));
        atomicMax(a.row_key + row, ((unsigned long long)key << 32) | (0xFFFFFFFFull - col));
    }
    if (bad) atomicOr(a.row_bad + row, 1u);
}

__global__ void __launch_bounds__(LM_NT, 1)
lm_head_kernel(const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap wmap, const LmArgs a) {
    extern __shared__ uint8_t lm_raw[];
    uint8_t* smem = lm_raw + ((1024u - (lm_s(lm_raw) & 1023u)) & 1023u);
    uint8_t* As = smem;
    uint8_t* Bs = smem + LM_ST * LM_ABYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + LM_ST * LM_BBYTES);
    uint64_t* full = bars;               // [LM_ST]
    uint64_t* empty = bars + LM_ST;      // [LM_ST]
    uint64_t* tfull = bars + 2 * LM_ST;  // [2]
    uint64_t* tempty = tfull + 2;        // [2]
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < LM_ST; ++s) {
            lm_init(full + s, 1);
            lm_init(empty + s, 1);
        }
        for (int i = 0; i < 2; ++i) {
            lm_init(tfull + i, 1);
            lm_init(tempty + i, 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(lm_s(tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    pdl_wait();
    const int n_mt = (a.rows + LM_BM - 1) / LM_BM, n_nt = (a.V + LM_BN - 1) / LM_BN;
    const int ntiles = n_mt * n_nt, nk = a.d / LM_BK;

    if (warp == 0) {
        if (lane == 0) {  // ================= TMA producer
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int mt = t % n_mt, nt = t / n_mt;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % LM_ST;
                    if (it >= LM_ST) lm_wait(empty + s, ((it / LM_ST) - 1) & 1);
                    lm_arrive_tx(full + s, LM_ABYTES + LM_BBYTES);
                    lm_tma(As + s * LM_ABYTES, &hmap, kb * LM_BK, mt * LM_BM, full + s);
                    lm_tma(Bs + s * LM_BBYTES, &wmap, kb * LM_BK, nt * LM_BN, full + s);
                }
            }
        }
    } else if (warp == 1) {  // ================= MMA issuer
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(LM_BN >> 3) << 17) |
                               ((uint32_t)(LM_BM >> 4) << 24);
        int it = 0, ti = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++ti) {
            const int ab = ti & 1;
            if (ti >= 2) lm_wait(tempty + ab, ((ti >> 1) - 1) & 1);  // the epilogue drained it
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            for (int kb = 0; kb < nk; ++kb, ++it) {
                const int s = it % LM_ST;
                lm_wait(full + s, (it / LM_ST) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (lane == 0) {
                    const uint32_t aa = lm_s(As + s * LM_ABYTES), ba = lm_s(Bs + s * LM_BBYTES);
#pragma unroll
                    for (int kk = 0; kk < LM_BK / 16; ++kk) {
                        const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
                        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                                     ::"r"(tmem + ab * LM_BN), "l"(lm_desc(aa + kk * 32)), "l"(lm_desc(ba + kk * 32)),
                                       "r"(idesc), "r"(acc) : "memory");
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                 ::"r"(lm_s(empty + s)) : "memory");
                    if (kb == nk - 1)
                        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                                     ::"r"(lm_s(tfull + ab)) : "memory");
                }
                __syncwarp();
            }
        }
    } else {  // ================= epilogue: warps 2-5, lane quarter (warp % 4)
        const int q = warp & 3;
        int ti = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++ti) {
            const int mt = t % n_mt, nt = t / n_mt;
            const int ab = ti & 1;
            lm_wait(tfull + ab, (ti >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int row = mt * LM_BM + q * 32 + lane;
            uint32_t best, bad;
            lm_drain(a, tmem + ((uint32_t)(q * 32) << 16) + ab * LM_BN, row, nt, best, bad);
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            lm_arrive(tempty + ab);  // this accumulator may be overwritten
            lm_stats(a, row, nt, best, bad);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
    __threadfence();
    pdl_trigger();
}

// ---- the CTA-pair kernel (default): tcgen05.mma.cta_group::2, 256 x 256 tiles per pair of SMs.
// CTA rank r of the pair holds rows [r*128, r*128+128) of the tile's A block and rows
// [r*128, r*128+128) of its W block (N half) at identical shared-memory offsets; the leader's
// single MMA (M 256, N 256, K 16) reads both halves of both operands and writes each CTA's 128
// accumulator rows into that CTA's TMEM.  Per SM this halves the W bytes staged per MMA (32 KB
// instead of 48 KB per K-block and SM), which relieves shared-memory bandwidth and the L2->SM
// traffic of the 1-CTA kernel above.  Both producers complete_tx on the LEADER's full barrier
// (cta_group::2 TMA); the leader's commits arrive on both CTAs' empty / tfull barriers
// (multicast); both CTAs' epilogue warps arrive on the leader's tempty barrier.
#ifndef BS_LM2_ST
#define BS_LM2_ST 6
#endif
constexpr int LM2_ST = BS_LM2_ST;
constexpr uint32_t LM2_HALF = 128 * LM_BK * 2;  // 16 KB: 128 rows x 64 bf16
constexpr size_t LM2_SMEM = 1024 + (size_t)LM2_ST * 2 * LM2_HALF + 256;

__device__ __forceinline__ uint32_t lm_mapa0(uint32_t saddr) {  // the leader CTA's copy of a shared address
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(saddr));
    return r;
}
__device__ __forceinline__ void lm_tma2(void* dst, const CUtensorMap* m, int x, int y, uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(lm_s(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void lm_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// a wait that acquires arrivals released at cluster scope (the peer CTA's epilogue)
__device__ __forceinline__ void lm_wait_cluster(uint64_t* b, uint32_t ph) {
    uint32_t ok = 0;
    uint64_t t0 = 0;
    for (int spin = 0; !ok; ++spin) {
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n"
                     "selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(lm_s(b)), "r"(ph), "r"(1000000u) : "memory");
        if (spin == 64) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        if (spin > 64 && (spin & 255) == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 2000000000ull) __trap();  // 2 s: protocol bug
        }
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(LM_NT, 1)
lm_head_pair_kernel(const __grid_constant__ CUtensorMap hmap, const __grid_constant__ CUtensorMap wmap,
                    const LmArgs a) {
    extern __shared__ uint8_t lm_raw[];
    uint8_t* smem = lm_raw + ((1024u - (lm_s(lm_raw) & 1023u)) & 1023u);
    uint8_t* As = smem;
    uint8_t* Bs = smem + LM2_ST * LM2_HALF;
    uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + LM2_ST * LM2_HALF);
    uint64_t* full = bars;                // [LM2_ST] (the leader's are used)
    uint64_t* empty = bars + LM2_ST;      // [LM2_ST]
    uint64_t* tfull = bars + 2 * LM2_ST;  // [2]
    uint64_t* tempty = tfull + 2;         // [2] (the leader's are used)
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        for (int s = 0; s < LM2_ST; ++s) {
            lm_init(full + s, 1);
            lm_init(empty + s, 1);
        }
        for (int i = 0; i < 2; ++i) {
            lm_init(tfull + i, 1);
            lm_init(tempty + i, 8);  // 4 epilogue warps x 2 CTAs
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // one warp of each CTA of the pair
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(lm_s(tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    lm_cluster_sync();  // both CTAs' barriers initialised and TMEM allocated
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tslot;
    pdl_wait();
    const int n_mp = (a.rows + 2 * LM_BM - 1) / (2 * LM_BM), n_nt = (a.V + LM_BN - 1) / LM_BN;
    const int ntiles = n_mp * n_nt, nk = a.d / LM_BK;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

    if (warp == 0) {
        if (lane == 0) {  // ================= TMA producer (both CTAs)
            const uint32_t full0 = lm_mapa0(lm_s(full));
            int it = 0;
            for (int t = pair; t < ntiles; t += npairs) {
                const int mp = t % n_mp, nt = t / n_mp;
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % LM2_ST;
                    if (it >= LM2_ST) lm_wait(empty + s, ((it / LM2_ST) - 1) & 1);
#ifdef BS_LM_EXP_NOLOAD  // measurement only: MMAs on stale tiles after the first ring fill
                    if (it >= LM2_ST) {
                        if (rank == 0) lm_arrive(full + s);
                        continue;
                    }
#endif
                    if (rank == 0) lm_arrive_tx(full + s, 4 * LM2_HALF);  // both CTAs' A and W halves
                    lm_tma2(As + s * LM2_HALF, &hmap, kb * LM_BK, mp * 2 * LM_BM + (int)rank * LM_BM, full0 + 8u * s);
                    lm_tma2(Bs + s * LM2_HALF, &wmap, kb * LM_BK, nt * LM_BN + (int)rank * (LM_BN / 2), full0 + 8u * s);
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {  // ================= MMA issuer (the leader CTA)
            const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(LM_BN >> 3) << 17) |
                                   ((uint32_t)((2 * LM_BM) >> 4) << 24);
            int it = 0, ti = 0;
            for (int t = pair; t < ntiles; t += npairs, ++ti) {
                const int ab = ti & 1;
                if (ti >= 2) lm_wait_cluster(tempty + ab, ((ti >> 1) - 1) & 1);  // both epilogues drained it
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                for (int kb = 0; kb < nk; ++kb, ++it) {
                    const int s = it % LM2_ST;
                    lm_wait(full + s, (it / LM2_ST) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    if (lane == 0) {
                        const uint32_t aa = lm_s(As + s * LM2_HALF), ba = lm_s(Bs + s * LM2_HALF);
#pragma unroll
                        for (int kk = 0; kk < LM_BK / 16; ++kk) {
                            const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
                            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                                         "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                                         ::"r"(tmem + ab * LM_BN), "l"(lm_desc(aa + kk * 32)), "l"(lm_desc(ba + kk * 32)),
                                           "r"(idesc), "r"(acc) : "memory");
                        }
                        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                                     ::"r"(lm_s(empty + s)), "h"((uint16_t)3) : "memory");
                        if (kb == nk - 1)
                            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                                         ::"r"(lm_s(tfull + ab)), "h"((uint16_t)3) : "memory");
                    }
                    __syncwarp();
                }
            }
        }
    } else {  // ================= epilogue: warps 2-5 of both CTAs, lane quarter (warp % 4)
        const int q = warp & 3;
        const uint32_t tempty0 = lm_mapa0(lm_s(tempty));
        int ti = 0;
        for (int t = pair; t < ntiles; t += npairs, ++ti) {
            const int mp = t % n_mp, nt = t / n_mp;
            const int ab = ti & 1;
            lm_wait(tfull + ab, (ti >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const int row = mp * 2 * LM_BM + (int)rank * LM_BM + q * 32 + lane;
            uint32_t best = 0, bad = 0;
#ifndef BS_LM_EXP_NOEPI  // measurement only: no drain
            lm_drain(a, tmem + ((uint32_t)(q * 32) << 16) + ab * LM_BN, row, nt, best, bad);
#endif
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0)  // this accumulator may be overwritten (the leader's barrier)
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty0 + 8u * ab)
                             : "memory");
            lm_stats(a, row, nt, best, bad);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    lm_cluster_sync();  // neither CTA frees TMEM (or exits) while the pair's MMAs / arrivals are in flight
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
    __threadfence();
    pdl_trigger();
}

static bool lm_map(CUtensorMap* m, const void* base, int64_t rows, int d, int box_rows) {
    // resolved once per process (a function-local static: thread-safe initialisation)
    static const PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        return (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
                qr == cudaDriverEntryPointSuccess)
                   ? reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p)
                   : nullptr;
    }();
    if (!enc) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)d * 2};
    const cuuint32_t box[2] = {(cuuint32_t)LM_BK, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace bs

extern "C" bs_status bs_lm_head_logits(const void* h, const void* w, int32_t rows, int32_t d, int32_t V, void* logits,
                                       int64_t ld_logits, uint64_t* row_key, uint32_t* row_bad, void* stream) {
    using namespace bs;
    if (!h || !w || !logits || !row_key || !row_bad || rows < 1 || V < 1 || d < LM_BK || d % LM_BK ||
        ld_logits < V || (((uintptr_t)h | (uintptr_t)w) & 15u))
        return BS_ERR_INVALID;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // the 1-CTA kernel (M 128 tiles) up to 128 rows, where the pair kernel's 256-row tiles would
    // be half padding (measured at d 3,584, V 151,936: 0.200 vs 0.233 ms at 128 rows, 86 vs 74 %
    // of HBM on W), the CTA-pair kernel above; BS_LM_KERNEL=1 / 2 forces one (measurement)
    static const int lm_kernel = [] {
        const char* e = getenv("BS_LM_KERNEL");
        return e ? atoi(e) : 0;
    }();
    const bool one_cta = lm_kernel == 1 || (lm_kernel != 2 && rows <= LM_BM);
    CUtensorMap hm, wm;
    if (!lm_map(&hm, h, rows, d, LM_BM) || !lm_map(&wm, w, V, d, one_cta ? LM_BN : LM_BN / 2)) return BS_ERR_CUDA;
    int dev = 0;
    cudaGetDevice(&dev);
    // per device: the smem attribute and the pair kernel's co-resident cluster count (a racing
    // second query is harmless)
    static std::atomic<int> configured[64] = {};
    static std::atomic<int> max_pairs[64] = {};
    if (dev < 0 || dev >= 64) return BS_ERR_CUDA;
    if (!configured[dev]) {
        if (cudaFuncSetAttribute(lm_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LM_SMEM) != cudaSuccess ||
            cudaFuncSetAttribute(lm_head_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LM2_SMEM) !=
                cudaSuccess)
            return BS_ERR_CUDA;
        cudaLaunchConfig_t qc = {};
        qc.gridDim = dim3(2);
        qc.blockDim = dim3(LM_NT);
        qc.dynamicSmemBytes = LM2_SMEM;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, lm_head_pair_kernel, &qc) != cudaSuccess || ncl < 1) return BS_ERR_CUDA;
        max_pairs[dev] = ncl;
        configured[dev] = 1;
    }
    if (cudaMemsetAsync(row_key, 0, sizeof(uint64_t) * (size_t)rows, st) != cudaSuccess ||
        cudaMemsetAsync(row_bad, 0, sizeof(uint32_t) * (size_t)rows, st) != cudaSuccess)
        return BS_ERR_CUDA;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    LmArgs a;
    a.rows = rows;
    a.d = d;
    a.V = V;
    a.logits = static_cast<uint16_t*>(logits);
    a.ld = ld_logits;
    a.row_key = reinterpret_cast<unsigned long long*>(row_key);
    a.row_bad = row_bad;
    cudaError_t e;
    if (one_cta) {
        const int ntiles = ((rows + LM_BM - 1) / LM_BM) * ((V + LM_BN - 1) / LM_BN);
        e = launch_pdl(lm_head_kernel, dim3(std::min(nsm, ntiles)), dim3(LM_NT), LM_SMEM, st, hm, wm, a);
    } else {
        const int ntiles = ((rows + 2 * LM_BM - 1) / (2 * LM_BM)) * ((V + LM_BN - 1) / LM_BN);
        const int pairs = std::min((int)max_pairs[dev], ntiles);
        e = launch_pdl(lm_head_pair_kernel, dim3(2 * pairs), dim3(LM_NT), LM2_SMEM, st, hm, wm, a);
    }
    return (e == cudaSuccess && cudaGetLastError() == cudaSuccess) ? BS_OK : BS_ERR_CUDA;
}
