// attn.cu — unified variable-query-length decode attention (Table 2
// at P:220-232): ONE launch serves plain decode requests (q_len = 1) and speculative requests
// (q_len = 1 + drafts) over a paged bf16 KV cache, with the short-query matmuls on the 5th-gen
// tensor cores ("the matrix multiplications for short-query verification are efficiently
// executed on tensor cores ... whose fixed tile sizes ensure negligible latency increase",
// P:250-251).  The work is HBM-bound on the KV stream; the tensor cores make the query length
// free up to the MMA's M = 128 rows.
//
// Design (sm_100a, one persistent CTA per SM, split-KV):
//  * work unit = (request b, KV head h, a range of 128-key tiles); its M = 128 rows are the
//    G = H_q / H_kv query heads of KV head h times the request's q_len query tokens
//    (row r = i * G + g; rows >= q_len * G are zero padding);
//  * warp 4 (one lane): TMA producer — each 128-key tile is 2 pages x 2 d-halves of K and of V,
//    eight 64 x 64 bf16 boxes (cp.async.bulk.tensor.2d, 128-byte swizzle) into a 2-stage ring;
//  * warp 5 (one lane): tcgen05 MMA issuer — S = Q K^T (M 128, N 128 keys, K 128 = d; A = Q in
//    smem, K-major; B = K tile, K-major) into TMEM columns [0, 128); after the softmax warps
//    wrote P, O_t = P V (N 128 = d, K 128 keys; A = P in smem, K-major; B = V tile, MN-major)
//    into TMEM columns [128, 256); tcgen05.commit arrives on mbarriers;
//  * warps 0-3 (thread = row = TMEM lane): online softmax in the exp2 domain with the causal
//    mask of the query block (token i at position ctx - q_len + i sees keys <= it), P -> bf16 in
//    swizzled smem, then O = O * alpha + O_t in registers; at the end of the unit the unnormalised
//    O, the running max m and sum l go to a per-unit partial;
//  * combine kernel: per (request, query head, token) the split partials are merged (the
//    flash-decoding rescale) into the bf16 output [T, H_q, d].
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/bubblespec.h"
#include "common.cuh"

namespace bs {

constexpr int AT_D = 128;        // head dim
constexpr int AT_PAGE = 64;      // tokens per KV page
constexpr int AT_TILE = 128;     // keys per tile (two pages)
constexpr int AT_ROWS = 128;     // MMA M
constexpr int AT_NT = 320;       // warps 0-7 softmax (two column groups), 8 TMA, 9 MMA
constexpr int AT_NSM = 256;      // softmax threads
constexpr int AT_KST = 2;  // K ring (a K tile is free once S = Q K^T completed)
constexpr int AT_VST = 3;  // V ring (a V tile is free once O += P V completed: later)
constexpr int AT_SPLIT_TILES = 16;  // tiles per work unit (2048 keys)
constexpr uint32_t AT_HALF = AT_ROWS * 128;          // one [128 rows][64 bf16] swizzled block: 16 KB
constexpr uint32_t AT_OP = 2 * AT_HALF;              // a 128 x 128 bf16 operand: 32 KB
constexpr size_t AT_SMEM = 1024 /*align*/ + (2 /*Q, P*/ + AT_KST + AT_VST) * (size_t)AT_OP + 256;

struct AttnUnit {
    int32_t b, h, t0, t1;
};

struct AttnArgs {
    const uint16_t* q;            // [T, H_q, d]
    const int32_t* page_table;    // [B, max_pages]
    int32_t max_pages;
    const int32_t* ctx_len;       // [B]
    const int32_t* q_off;         // [B + 1]
    const AttnUnit* units;
    int32_t n_units;
    int32_t H_q, H_kv, G;
    float c;                      // scale * log2(e)
    int64_t kv_rows;              // num_pages * H_kv * PAGE (tensor-map rows)
    float* part_o;                // [n_units, 128, d] unnormalised O
    float* part_ml;               // [n_units, 128, 2] (m, l) in the exp2 domain
};

// --------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void at_mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void at_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void at_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t at_now() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void at_wait(uint64_t* bar, uint32_t phase) {
    uint32_t ok = 0;
    uint64_t t0 = 0;
    for (int spin = 0; !ok; ++spin) {
        if (spin == 64) t0 = at_now();
        if (spin > 64 && (spin & 255) == 0 && at_now() - t0 > 2000000000ull) __trap();  // 2 s: protocol bug
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(phase), "r"(1000000u)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
        ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
// 32 lanes x 32 columns of 32 bits: thread = lane, v[j] = column col + j
__device__ __forceinline__ void tc_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

__device__ __forceinline__ void tc_st32(uint32_t taddr, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
        ::"r"(taddr), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
          "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]),
          "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]),
          "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2 (P is rounded to bf16 afterwards)
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Shared-memory matrix descriptor (tcgen05), 128-byte swizzle: start, leading / stride byte
// offsets (16-byte units), version 1, layout type 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor, kind::f16: D f32, A/B bf16, A K-major, B K- or MN-major, N, M = 128.
__host__ __device__ constexpr uint32_t f16_idesc(int N, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(AT_ROWS >> 4) << 24);
}

// Byte offset of element (row, k) (k in [0, 128)) in a 128 x 128 bf16 K-major operand stored as
// two swizzled [128 rows][64] halves: 16-byte chunk u of a row lands at chunk u ^ (row & 7).
__device__ __forceinline__ uint32_t sw_off(int row, int k) {
    const int half = k >> 6, u = (k & 63) >> 3;
    return (uint32_t)half * AT_HALF + (uint32_t)row * 128u + (uint32_t)((u ^ (row & 7)) << 4) + (uint32_t)((k & 7) * 2);
}

__global__ void __launch_bounds__(AT_NT, 1)
unified_attn_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                    const AttnArgs a) {
    extern __shared__ uint8_t at_smem_raw[];
    const uint32_t raw = smem_u32(at_smem_raw);
    uint8_t* smem = at_smem_raw + ((1024u - (raw & 1023u)) & 1023u);  // 1024-byte aligned (swizzle atoms)
    uint8_t* Qs = smem;
    uint8_t* Ps = smem + AT_OP;
    uint8_t* Ks = smem + 2 * AT_OP;           // K stage s at s * OP
    uint8_t* Vs = Ks + AT_KST * AT_OP;        // V stage s at s * OP
    uint64_t* bars = reinterpret_cast<uint64_t*>(Vs + AT_VST * AT_OP);
    uint64_t* k_full = bars;                  // [AT_KST]
    uint64_t* k_empty = bars + AT_KST;        // [AT_KST]
    uint64_t* v_full = bars + 2 * AT_KST;     // [AT_VST]
    uint64_t* v_empty = v_full + AT_VST;      // [AT_VST]
    uint64_t* s_full = v_empty + AT_VST;      // [2]: S double-buffered in TMEM
    uint64_t* p_full = s_full + 2;
    uint64_t* o_full = s_full + 3;
    uint64_t* q_full = s_full + 4;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 5);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < AT_KST; ++s) {
            at_mbar_init(k_full + s, 1);
            at_mbar_init(k_empty + s, 1);
        }
        for (int s = 0; s < AT_VST; ++s) {
            at_mbar_init(v_full + s, 1);
            at_mbar_init(v_empty + s, 1);
        }
        at_mbar_init(s_full, 1);
        at_mbar_init(s_full + 1, 1);
        at_mbar_init(p_full, AT_NSM);
        at_mbar_init(o_full, 1);
        at_mbar_init(q_full, AT_NSM);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 9) {  // TMEM: S in columns [0, 128) and [128, 256) (alternating tiles), O in [256, 384)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                     ::"r"(smem_u32(tmem_slot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();

    if (warp == 8) {
        // ================================================================ TMA producer
        if (lane == 0) {
            int it = 0;
            for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
                const AttnUnit un = a.units[u];
                const int ctx = a.ctx_len[un.b];
                const int npg = (ctx + AT_PAGE - 1) / AT_PAGE;
                for (int t = un.t0; t < un.t1; ++t, ++it) {
                    const int ks = it % AT_KST, vs = it % AT_VST;
                    long long row[2];
#pragma unroll
                    for (int pg = 0; pg < 2; ++pg) {
                        const int pi = 2 * t + pg;
                        // a page past the context: rows beyond the tensor map -> TMA zero fill
                        row[pg] = (pi < npg)
                            ? ((long long)a.page_table[(long long)un.b * a.max_pages + pi] * a.H_kv + un.h) * AT_PAGE
                            : a.kv_rows;
                    }
                    if (it >= AT_KST) at_wait(k_empty + ks, ((it / AT_KST) - 1) & 1);
                    at_arrive_tx(k_full + ks, AT_OP);
#pragma unroll
                    for (int pg = 0; pg < 2; ++pg)
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf)
                            tma_load_2d(Ks + ks * AT_OP + hf * AT_HALF + pg * (AT_PAGE * 128), &kmap, hf * 64,
                                        (int)row[pg], k_full + ks);
                    if (it >= AT_VST) at_wait(v_empty + vs, ((it / AT_VST) - 1) & 1);
                    at_arrive_tx(v_full + vs, AT_OP);
#pragma unroll
                    for (int pg = 0; pg < 2; ++pg)
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf)
                            tma_load_2d(Vs + vs * AT_OP + hf * AT_HALF + pg * (AT_PAGE * 128), &vmap, hf * 64,
                                        (int)row[pg], v_full + vs);
                }
            }
        }
    } else if (warp == 9) {
        // ================================================================ MMA issuer
        const uint32_t id1 = f16_idesc(AT_TILE, false), id2 = f16_idesc(AT_D, true);
        const uint32_t qa = smem_u32(Qs), pa = smem_u32(Ps);
        // O_t = P V for tile j (its P is in smem once p_full completes), then release the stage
        auto mma2 = [&](int j, bool acc_prev) {
            at_wait(v_full + j % AT_VST, (j / AT_VST) & 1);
            at_wait(p_full, j & 1);
            tc_fence_after();
            const uint32_t va = smem_u32(Vs + (j % AT_VST) * AT_OP);
            if (lane == 0) {
#pragma unroll
                for (int kk = 0; kk < AT_TILE / 16; ++kk) {  // K dimension = keys
                    const uint32_t aoff = (uint32_t)(kk >> 2) * AT_HALF + (uint32_t)(kk & 3) * 32u;
                    // V: MN-major (d contiguous), 16 keys = 2048 bytes; d-halves 16 KB apart
                    tc_mma(tmem + 256, sw128_desc(pa + aoff, 16, 1024), sw128_desc(va + kk * 2048u, AT_HALF, 1024),
                           id2, (acc_prev || kk > 0) ? 1u : 0u);  // O accumulates in TMEM over the unit
                }
                tc_commit(o_full);
                tc_commit(v_empty + j % AT_VST);
            }
            __syncwarp();
        };
        int it = 0, uq = 0;
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x, ++uq) {
            const AttnUnit un = a.units[u];
            at_wait(q_full, uq & 1);  // this unit's Q rows are in smem
            tc_fence_after();
            for (int t = un.t0; t < un.t1; ++t, ++it) {
                // S(t) = Q K^T into the S buffer of tile parity: issued before the previous tile's
                // P V, so it runs while the softmax warps still work on the previous tile
                const int ks = it % AT_KST;
                at_wait(k_full + ks, (it / AT_KST) & 1);
                tc_fence_after();
                const uint32_t ka = smem_u32(Ks + ks * AT_OP);
                if (lane == 0) {
#pragma unroll
                    for (int kk = 0; kk < AT_D / 16; ++kk) {  // K dimension = d
                        const uint32_t off = (uint32_t)(kk >> 2) * AT_HALF + (uint32_t)(kk & 3) * 32u;
                        tc_mma(tmem + (it & 1) * 128, sw128_desc(qa + off, 16, 1024), sw128_desc(ka + off, 16, 1024),
                               id1, kk > 0);
                    }
                    tc_commit(s_full + (it & 1));
                    tc_commit(k_empty + ks);
                }
                __syncwarp();
                if (t > un.t0) mma2(it - 1, t - 1 > un.t0);
            }
            mma2(it - 1, un.t1 - 1 > un.t0);
        }
    } else {
        // ================================================================ softmax / correction
        // Two column groups share each row (warps w and w + 4 see the same TMEM lanes): group
        // grp reads S columns / writes P for keys [64 grp, 64 grp + 64) and owns O columns
        // [64 grp, 64 grp + 64); the two halves of the row max meet in shared memory.  O
        // accumulates in TMEM across the unit's tiles (MMA accumulate); the running max used for
        // the exponent is raised only when the true max exceeds it by more than 2^8 (then O and
        // l are rescaled in place), so most tiles touch O not at all.
        __shared__ float l_other[AT_ROWS];
        __shared__ float pmax[2][AT_ROWS];  // [group][row]; a pair barrier before each write keeps
                                            // the partner's read of the previous tile's value first
        const int grp = warp >> 2;
        const int r = (warp & 3) * 32 + lane;  // row = TMEM lane
        const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        constexpr float RESCALE = 8.f;  // log2 headroom of the stale max
        int it = 0, uq = 0;
        for (int u = blockIdx.x; u < a.n_units; u += gridDim.x, ++uq) {
            const AttnUnit un = a.units[u];
            const int ctx = a.ctx_len[un.b];
            const int q0 = a.q_off[un.b], ql = a.q_off[un.b + 1] - q0;
            const int nrows = ql * a.G;
            const int qi = r / a.G, g = r - qi * a.G;
            const int pos = ctx - ql + qi;  // absolute position of this row's query token
            const int full_below = ctx - ql;  // keys < = this are visible to every row
            // this group's half of the Q row -> swizzled smem (zero padding rows); the previous
            // unit's MMAs are complete
            {
                const uint4* src = reinterpret_cast<const uint4*>(a.q + ((long long)(q0 + qi) * a.H_q + un.h * a.G + g) * AT_D);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int cc = grp * 8 + c;
                    const uint4 v = (r < nrows) ? __ldg(src + cc) : make_uint4(0, 0, 0, 0);
                    *reinterpret_cast<uint4*>(Qs + sw_off(r, cc * 8)) = v;
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            at_arrive(q_full);
            float m = -INFINITY, l = 0.f;
            for (int t = un.t0; t < un.t1; ++t, ++it) {
                at_wait(s_full + (it & 1), (it >> 1) & 1);
                tc_fence_after();
                const uint32_t srow = trow + (it & 1) * 128;
                const int key0 = t * AT_TILE + grp * 64;
                const bool edge = t * AT_TILE + AT_TILE - 1 > full_below;  // uniform over the CTA
                float sv[64];
                tc_ld32(srow + grp * 64, sv);
                tc_ld32(srow + grp * 64 + 32, sv + 32);
                float mx = -INFINITY;
                if (edge) {
#pragma unroll
                    for (int j = 0; j < 64; ++j) {
                        if (key0 + j > pos || key0 + j >= ctx) sv[j] = -INFINITY;
                        mx = fmaxf(mx, sv[j]);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 64; ++j) mx = fmaxf(mx, sv[j]);
                }
                asm volatile("bar.sync %0, 64;" ::"r"(2 + (warp & 3)) : "memory");  // partner read the last one
                pmax[grp][r] = mx;
                asm volatile("bar.sync %0, 64;" ::"r"(2 + (warp & 3)) : "memory");  // the row's two warps
                mx = fmaxf(mx, pmax[grp ^ 1][r]) * a.c;  // (c > 0)
                bool rescale = false;
                float alpha = 1.f;
                if (m == -INFINITY) {
                    m = mx;  // first visible keys of this row in the unit (O holds only zeros)
                } else if (mx > m + RESCALE) {
                    alpha = ex2(m - mx);
                    rescale = true;
                    m = mx;
                    l *= alpha;
                }
                // the previous tile's P V has landed in O (and no longer reads P): rescale O if
                // needed, then overwrite P
                if (t > un.t0) {  // the previous tile's P V has landed in O: rescale it if needed
                    at_wait(o_full, (it - 1) & 1);
                    tc_fence_after();
                    if (__any_sync(0xFFFFFFFFu, rescale)) {  // (tcgen05.ld/st are warp-collective)
#pragma unroll
                        for (int c2 = 0; c2 < 2; ++c2) {
                            float ov[32];
                            tc_ld32(trow + 256 + grp * 64 + c2 * 32, ov);
#pragma unroll
                            for (int j = 0; j < 32; ++j) ov[j] *= alpha;
                            tc_st32(trow + 256 + grp * 64 + c2 * 32, ov);
                        }
                    }
                }
                const float mneg = -m;
                const bool live = m != -INFINITY;
                float lt = 0.f;
#pragma unroll
                for (int j = 0; j < 64; j += 8) {  // P -> bf16, 16-byte swizzled stores
                    uint32_t w[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float p0 = live ? ex2(fmaf(sv[j + 2 * e], a.c, mneg)) : 0.f;
                        const float p1 = live ? ex2(fmaf(sv[j + 2 * e + 1], a.c, mneg)) : 0.f;
                        const __nv_bfloat162 pb = __floats2bfloat162_rn(p0, p1);
                        // the sum uses the bf16 values the MMA multiplies (P and l consistent)
                        const float2 pf = __bfloat1622float2(pb);
                        lt += pf.x + pf.y;
                        w[e] = *reinterpret_cast<const uint32_t*>(&pb);
                    }
                    *reinterpret_cast<uint4*>(Ps + sw_off(r, grp * 64 + j)) = make_uint4(w[0], w[1], w[2], w[3]);
                }
                l += lt;
                // keys past the context in this tile: zero their V rows (the cache may hold
                // anything there; 0 * NaN would poison O).  Row r of the tile = key
                // t * 128 + r; group grp zeroes d-half grp.
                if (t * AT_TILE + AT_TILE > ctx && t * AT_TILE + r >= ctx) {
                    at_wait(v_full + it % AT_VST, (it / AT_VST) & 1);  // V(t) has landed
                    uint8_t* Vt = Vs + (it % AT_VST) * AT_OP + grp * AT_HALF;
#pragma unroll
                    for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(Vt + r * 128 + c * 16) = make_uint4(0, 0, 0, 0);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tc_fence_before();
                at_arrive(p_full);
            }
            at_wait(o_full, (it - 1) & 1);  // the unit's last P V
            tc_fence_after();
            // the row sum is split over the two groups' keys
            if (grp == 1) l_other[r] = l;
            asm volatile("bar.sync 1, %0;" ::"n"(AT_NSM) : "memory");
            {
                float ov[64];  // (warp-collective loads, then the row's own stores)
                tc_ld32(trow + 256 + grp * 64, ov);
                tc_ld32(trow + 256 + grp * 64 + 32, ov + 32);
                if (r < nrows) {
                    float4* dst = reinterpret_cast<float4*>(a.part_o + ((long long)u * AT_ROWS + r) * AT_D + grp * 64);
#pragma unroll
                    for (int j = 0; j < 16; ++j) dst[j] = make_float4(ov[4 * j], ov[4 * j + 1], ov[4 * j + 2], ov[4 * j + 3]);
                    if (grp == 0) {
                        a.part_ml[((long long)u * AT_ROWS + r) * 2] = m;
                        a.part_ml[((long long)u * AT_ROWS + r) * 2 + 1] = l + l_other[r];
                    }
                }
            }
            tc_fence_before();
            asm volatile("bar.sync 1, %0;" ::"n"(AT_NSM) : "memory");  // l_other reused next unit
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
    __threadfence();
    pdl_trigger();
}

// Merge the split partials of every (request, query head, token) row: one warp per row, lane
// owns 4 of the d = 128 outputs.
__global__ void __launch_bounds__(256) attn_combine_kernel(const AttnArgs a, const int32_t* row_b,
                                                           const int32_t* bh_unit0, const int32_t* bh_units,
                                                           uint16_t* out, int32_t n_rows) {
    pdl_wait();
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n_rows) return;
    // w enumerates (token row tr of the batch, query head hq): tr = w / H_q
    const int tr = w / a.H_q, hq = w - tr * a.H_q;
    const int b = row_b[tr];
    const int i = tr - a.q_off[b];
    const int h = hq / a.G, g = hq - h * a.G;
    const int r = i * a.G + g;
    const int bh = b * a.H_kv + h;
    const int u0 = bh_unit0[bh], nu = bh_units[bh];
    float M = -INFINITY;
    for (int s = 0; s < nu; ++s) M = fmaxf(M, a.part_ml[((long long)(u0 + s) * AT_ROWS + r) * 2]);
    float acc[4] = {0.f, 0.f, 0.f, 0.f}, L = 0.f;
    for (int s = 0; s < nu; ++s) {
        const long long pr = (long long)(u0 + s) * AT_ROWS + r;
        const float ms = a.part_ml[pr * 2];
        if (ms == -INFINITY) continue;
        const float f = exp2f(ms - M);
        L = fmaf(a.part_ml[pr * 2 + 1], f, L);
        const float4 v = reinterpret_cast<const float4*>(a.part_o + pr * AT_D)[lane];
        acc[0] = fmaf(v.x, f, acc[0]);
        acc[1] = fmaf(v.y, f, acc[1]);
        acc[2] = fmaf(v.z, f, acc[2]);
        acc[3] = fmaf(v.w, f, acc[3]);
    }
    const float inv = 1.f / L;
    const __nv_bfloat162 lo = __floats2bfloat162_rn(acc[0] * inv, acc[1] * inv);
    const __nv_bfloat162 hi = __floats2bfloat162_rn(acc[2] * inv, acc[3] * inv);
    uint2 pk;
    pk.x = *reinterpret_cast<const uint32_t*>(&lo);
    pk.y = *reinterpret_cast<const uint32_t*>(&hi);
    reinterpret_cast<uint2*>(out + ((long long)tr * a.H_q + hq) * AT_D)[lane] = pk;
    __threadfence();
    pdl_trigger();
}

// Device twin of workloads/attn.py _vals (synthetic inputs, NOT the method): value i =
// (sum of the 4 bytes of h32(i * 0x9E3779B1 + base) - 510) * mult, rounded to bf16.
__global__ void synth_attn_kernel(uint16_t* out, int64_t n, uint32_t base, float mult) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t h = h32((uint32_t)i * 0x9E3779B1u + base);
        const int s = (int)(h & 255u) + (int)((h >> 8) & 255u) + (int)((h >> 16) & 255u) + (int)(h >> 24) - 510;
        const __nv_bfloat16 bv = __float2bfloat16_rn((float)s * mult);
        out[i] = *reinterpret_cast<const uint16_t*>(&bv);
    }
}

// --------------------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn() {
    // resolved once per process (a function-local static: thread-safe initialisation)
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        return (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                   ? reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p)
                   : nullptr;
    }();
    return fn;
}

static bool make_kv_map(CUtensorMap* map, const void* base, int64_t rows) {
    auto enc = tmap_encode_fn();
    if (!enc) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)AT_D, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)AT_D * 2};
    const cuuint32_t box[2] = {64, AT_PAGE};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct AttnPlan {
    std::vector<AttnUnit> units;
    std::vector<int32_t> q_off, row_b, bh_unit0, bh_units;
};

static AttnPlan plan_attn(int B, const int32_t* ctx_len, const int32_t* q_len, int H_kv) {
    AttnPlan p;
    p.q_off.assign(B + 1, 0);
    for (int b = 0; b < B; ++b) p.q_off[b + 1] = p.q_off[b] + q_len[b];
    p.row_b.resize(p.q_off[B]);
    for (int b = 0; b < B; ++b)
        for (int i = p.q_off[b]; i < p.q_off[b + 1]; ++i) p.row_b[i] = b;
    p.bh_unit0.resize((size_t)B * H_kv);
    p.bh_units.resize((size_t)B * H_kv);
    for (int b = 0; b < B; ++b) {
        const int ntile = (ctx_len[b] + AT_TILE - 1) / AT_TILE;
        const int nsplit = std::max(1, (ntile + AT_SPLIT_TILES - 1) / AT_SPLIT_TILES);
        for (int h = 0; h < H_kv; ++h) {
            p.bh_unit0[(size_t)b * H_kv + h] = (int32_t)p.units.size();
            p.bh_units[(size_t)b * H_kv + h] = nsplit;
            for (int s = 0; s < nsplit; ++s) {
                const int t0 = (int)((long long)ntile * s / nsplit), t1 = (int)((long long)ntile * (s + 1) / nsplit);
                p.units.push_back({b, h, t0, t1});
            }
        }
    }
    return p;
}

// Workspace layout: units | q_off | ctx_len copy not needed (device input) | row_b | bh_unit0 |
// bh_units | part_ml | part_o (each region 256-byte aligned).
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
static size_t ws_bytes(const AttnPlan& p) {
    size_t n = 0;
    n += align256(p.units.size() * sizeof(AttnUnit));
    n += align256(p.q_off.size() * 4) + align256(p.row_b.size() * 4) + 2 * align256(p.bh_unit0.size() * 4);
    n += align256(p.units.size() * AT_ROWS * 2 * 4);
    n += align256(p.units.size() * AT_ROWS * (size_t)AT_D * 4);
    return n;
}

}  // namespace bs

extern "C" {

bs_status bsx_synth_attn_values(void* out, int64_t n, uint32_t base, float mult, void* stream) {
    if (!out || n < 0) return BS_ERR_INVALID;
    if (n == 0) return BS_OK;
    const int grid = (int)std::min<int64_t>(4096, (n + 255) / 256);
    bs::synth_attn_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<uint16_t*>(out), n, base,
                                                                                 mult);
    return cudaGetLastError() == cudaSuccess ? BS_OK : BS_ERR_CUDA;
}

bs_status bs_unified_attention_workspace(int32_t B, const int32_t* ctx_len, const int32_t* q_len, int32_t H_q,
                                         int32_t H_kv, int64_t* bytes) {
    if (B < 1 || !ctx_len || !q_len || !bytes || H_kv < 1 || H_q < H_kv || H_q % H_kv) return BS_ERR_INVALID;
    *bytes = (int64_t)bs::ws_bytes(bs::plan_attn(B, ctx_len, q_len, H_kv));
    return BS_OK;
}

bs_status bs_unified_attention(const void* q, const void* k_cache, const void* v_cache, int64_t num_pages,
                               const int32_t* page_table, int32_t max_pages, const int32_t* ctx_len_dev,
                               const int32_t* ctx_len, const int32_t* q_len, int32_t B, int32_t H_q, int32_t H_kv,
                               int32_t head_dim, int32_t page_size, float scale, void* out, void* workspace,
                               int64_t workspace_bytes, void* stream) {
    using namespace bs;
    if (!q || !k_cache || !v_cache || !page_table || !ctx_len_dev || !ctx_len || !q_len || !out || !workspace)
        return BS_ERR_INVALID;
    if (head_dim != AT_D || page_size != AT_PAGE || B < 1 || H_kv < 1 || H_q % H_kv || num_pages < 1)
        return BS_ERR_INVALID;
    const int G = H_q / H_kv;
    for (int b = 0; b < B; ++b) {
        if (q_len[b] < 1 || ctx_len[b] < q_len[b] || q_len[b] * G > AT_ROWS) return BS_ERR_INVALID;
        if ((ctx_len[b] + AT_PAGE - 1) / AT_PAGE > max_pages) return BS_ERR_INVALID;
    }
    const int64_t kv_rows = num_pages * H_kv * AT_PAGE;
    if (kv_rows >= (1ll << 31)) return BS_ERR_INVALID;
    const AttnPlan p = plan_attn(B, ctx_len, q_len, H_kv);
    if ((int64_t)ws_bytes(p) > workspace_bytes) return BS_ERR_CAPACITY;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* w = static_cast<uint8_t*>(workspace);
    cudaError_t put_err = cudaSuccess;
    auto put = [&](const void* src, size_t bytes) {
        uint8_t* d = w;
        w += align256(bytes);
        // pageable source: the runtime stages it before returning, so the host plan may go
        if (bytes && put_err == cudaSuccess) put_err = cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st);
        return d;
    };
    AttnArgs a = {};
    a.units = reinterpret_cast<const AttnUnit*>(put(p.units.data(), p.units.size() * sizeof(AttnUnit)));
    a.q_off = reinterpret_cast<const int32_t*>(put(p.q_off.data(), p.q_off.size() * 4));
    const int32_t* row_b = reinterpret_cast<const int32_t*>(put(p.row_b.data(), p.row_b.size() * 4));
    const int32_t* u0 = reinterpret_cast<const int32_t*>(put(p.bh_unit0.data(), p.bh_unit0.size() * 4));
    const int32_t* un = reinterpret_cast<const int32_t*>(put(p.bh_units.data(), p.bh_units.size() * 4));
    if (put_err != cudaSuccess) return BS_ERR_CUDA;
    a.part_ml = reinterpret_cast<float*>(w);
    w += align256(p.units.size() * AT_ROWS * 2 * 4);
    a.part_o = reinterpret_cast<float*>(w);
    a.q = static_cast<const uint16_t*>(q);
    a.page_table = page_table;
    a.max_pages = max_pages;
    a.ctx_len = ctx_len_dev;
    a.n_units = (int32_t)p.units.size();
    a.H_q = H_q;
    a.H_kv = H_kv;
    a.G = G;
    a.c = (scale > 0.f ? scale : 1.f / sqrtf((float)AT_D)) * 1.4426950408889634f;
    a.kv_rows = kv_rows;
    CUtensorMap km, vm;
    if (!make_kv_map(&km, k_cache, kv_rows) || !make_kv_map(&vm, v_cache, kv_rows)) return BS_ERR_CUDA;
    int dev = 0;
    cudaGetDevice(&dev);
    // per-device launch attribute (setting it twice from racing threads is harmless)
    static std::atomic<int> configured[64] = {};
    if (dev < 0 || dev >= 64 || !configured[dev]) {
        if (cudaFuncSetAttribute(unified_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)AT_SMEM) !=
            cudaSuccess)
            return BS_ERR_CUDA;
        if (dev >= 0 && dev < 64) configured[dev] = 1;
    }
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min(nsm, a.n_units);
    cudaError_t e = launch_pdl(unified_attn_kernel, dim3(grid), dim3(AT_NT), AT_SMEM, st, km, vm, a);
    if (e != cudaSuccess) return BS_ERR_CUDA;
    const int n_rows = p.q_off[B] * H_q;
    e = launch_pdl(attn_combine_kernel, dim3((n_rows * 32 + 255) / 256), dim3(256), 0, st, a, row_b, u0, un,
                   static_cast<uint16_t*>(out), (int32_t)n_rows);
    if (e != cudaSuccess) return BS_ERR_CUDA;
    return cudaGetLastError() == cudaSuccess ? BS_OK : BS_ERR_CUDA;
}

}  // extern "C"
