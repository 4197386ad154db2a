// lmhead.cu — the LM-head GEMM with the verify's first pass fused into its epilogue (SURVEY
// §8(f)3).  logits[r, v] = bf16(sum_k h[r, k] W[v, k]) on the 5th-gen tensor cores, and, while the
// accumulator tile is in registers, the row statistics the verify's max pass computes (readings
// R0/R1: the row maximum of the bf16 logits, the lowest index attaining it, and whether a NaN /
// +inf occurs), folded across the N tiles with one 64-bit atomicMax per (row, tile).  A verify
// launch given those statistics (bsx_set_row_stats) skips its max pass: every CTA of a row's
// cluster publishes the row's precomputed maximum.  (An exact verify cannot also skip the logits
// round trip: its integer masses need the row maximum before any mass.)
//
// Kernel (sm_100a, one persistent CTA per SM): 128 x 256 output tiles, M fastest so the CTAs
// working at one time share the W tile through L2; warp 0 issues TMA loads (128-byte swizzle,
// K-blocks of 64) into a 4-stage ring; warp 1 issues tcgen05.mma kind::f16 (M 128, N 256, K 16)
// into one of two TMEM accumulators (2 x 256 columns); warps 2-5 drain the other accumulator
// (tcgen05.ld, fp32 -> bf16 round-to-nearest-even, global stores, row statistics).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdint>

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
// bf16 bits -> 16-bit key ordered like the values (NaN excluded by the caller)
__device__ __forceinline__ uint32_t lm_key(uint32_t b) { return (b & 0x8000u) ? (~b & 0xFFFFu) : (b | 0x8000u); }

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
            const bool rok = row < a.rows;
            uint32_t best = 0;  // (key << 16 | ~col) over this tile, 0 = none
            uint32_t bad = 0;
            uint16_t* dst = a.logits + (int64_t)(rok ? row : 0) * a.ld + (int64_t)nt * LM_BN;
#pragma unroll 1
            for (int c = 0; c < LM_BN / 32; ++c) {
                uint32_t r[32];
                lm_ld32(tmem + ((uint32_t)(q * 32) << 16) + ab * LM_BN + c * 32, r);
                const int col0 = nt * LM_BN + c * 32;
                uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const __nv_bfloat162 p2 = __floats2bfloat162_rn(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
                    pk[j] = *reinterpret_cast<const uint32_t*>(&p2);
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const uint32_t b = (j & 1) ? (pk[j >> 1] >> 16) : (pk[j >> 1] & 0xFFFFu);
                    const int col = col0 + j;
                    if (col < a.V) {
                        if ((b & 0x7FFFu) >= 0x7F80u && b != 0xFF80u) {  // NaN or +inf (R0)
                            bad |= ((b & 0x7FFFu) > 0x7F80u || b == 0x7F80u) ? 1u : 0u;
                            if ((b & 0x7FFFu) > 0x7F80u) continue;  // NaN: not a maximum
                        }
                        const uint32_t kv = (lm_key(b) << 16) | (0xFFFFu - (uint32_t)(c * 32 + j));
                        best = max(best, kv);
                    }
                }
                if (rok) {
                    if (col0 + 32 <= a.V && (((uintptr_t)(dst + c * 32) & 15u) == 0)) {
                        uint4* d4 = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
                        for (int j = 0; j < 4; ++j) d4[j] = make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
                    } else {
                        for (int j = 0; j < 32 && col0 + j < a.V; ++j)
                            dst[c * 32 + j] = (uint16_t)((j & 1) ? (pk[j >> 1] >> 16) : (pk[j >> 1] & 0xFFFFu));
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            lm_arrive(tempty + ab);  // this accumulator may be overwritten
            if (rok) {
                if (best) {
                    const uint32_t key = best >> 16, col = (uint32_t)nt * LM_BN + (0xFFFFu - (best & 0xFFFFu));
                    atomicMax(a.row_key + row, ((unsigned long long)key << 32) | (0xFFFFFFFFull - col));
                }
                if (bad) atomicOr(a.row_bad + row, 1u);
            }
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
    CUtensorMap hm, wm;
    if (!lm_map(&hm, h, rows, d, LM_BM) || !lm_map(&wm, w, V, d, LM_BN)) return BS_ERR_CUDA;
    int dev = 0;
    cudaGetDevice(&dev);
    static std::atomic<int> configured[64] = {};  // per-device attribute (a racing second set is harmless)
    if (dev < 0 || dev >= 64 || !configured[dev]) {
        if (cudaFuncSetAttribute(lm_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LM_SMEM) != cudaSuccess)
            return BS_ERR_CUDA;
        if (dev >= 0 && dev < 64) configured[dev] = 1;
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
    const int ntiles = ((rows + LM_BM - 1) / LM_BM) * ((V + LM_BN - 1) / LM_BN);
    cudaError_t e = launch_pdl(lm_head_kernel, dim3(std::min(nsm, ntiles)), dim3(LM_NT), LM_SMEM, st, hm, wm, a);
    return (e == cudaSuccess && cudaGetLastError() == cudaSuccess) ? BS_OK : BS_ERR_CUDA;
}
