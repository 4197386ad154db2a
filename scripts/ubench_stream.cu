// Streaming skeleton of a cluster verify pipeline (no scheduler): each cluster streams a
// static list of logits rows; per CTA a slice of every row goes HBM -> shared memory (one
// bulk copy), max warps reduce it, the cluster max travels by DSMEM st.async, mass warps
// compute the exact integer masses of reading R (no per-row barrier between mass warps),
// the epilogue warp combines the per-warp sums and exchanges slice sums.  Measures the raw
// row throughput of (cluster size, buffers, CTAs per SM, warps) configurations.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_08862_b200/csrc -o /tmp/ubs scripts/ubench_stream.cu
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"
#include "verify_math.cuh"

using namespace bs;
namespace cg = cooperative_groups;

constexpr int TILE = 512;
constexpr int MAXT = 160;

template <int CL, int NB>
struct Sh {
    uint64_t full[NB], empty[NB];
    uint64_t maxbar[2 * NB], sumbar[2 * NB], sumready[2 * NB], eempty[2 * NB];
    uint4 cmax[2 * NB][CL];
    uint4 csum[2 * NB][CL];
    unsigned long long wsum[2 * NB][20];
    float wmax[8];
};


// ---- mass-loop variants (exact reading R, bit-identical results)
// bf16 unpack on the ALU pipe (PRMT / LOP3 instead of IMAD.U32)
__device__ __forceinline__ float lo_alu(uint32_t w) { return __uint_as_float(__byte_perm(w, 0u, 0x1044u)); }
__device__ __forceinline__ float hi_alu(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t shl23_alu(uint32_t t) {
    uint32_t r;
    asm("shf.l.wrap.b32 %0, %1, %2, 23;" : "=r"(r) : "r"(0u), "r"(t));
    return r;
}
__device__ __forceinline__ uint32_t add_alu(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// w is already clamped from below in bf16 (HMNMX2 with the row's L0): no y clamp
__device__ __forceinline__ void pair_core(uint32_t w, float c, float nmc, float magic, F2& t, F2& p) {
    const F2 l{lo_alu(w), hi_alu(w)};
    const F2 y = ffma2(l, F2{c, c}, F2{nmc, nmc});
    t = fadd2(y, F2{magic, magic});
    const F2 n = fadd2(t, F2{-magic, -magic});
    const F2 f = fadd2(y, F2{-n.x, -n.y});
    p = ffma2(F2{BS_C5, BS_C5}, f, F2{BS_C4, BS_C4});
    p = ffma2(p, f, F2{BS_C3, BS_C3});
    p = ffma2(p, f, F2{BS_C2, BS_C2});
    p = ffma2(p, f, F2{BS_C1, BS_C1});
    p = ffma2(p, f, F2{BS_C0, BS_C0});
}
__device__ __forceinline__ void pair_core_s(uint32_t w, float c, float nmc, float magic, F2& t, F2& p) {
    const F2 l{lo_alu(w), hi_alu(w)};
    const F2 y = ffma2(l, F2{c, c}, F2{nmc, nmc});
    t = fadd2(y, F2{magic, magic});
    const F2 n = fadd2(t, F2{-magic, -magic});
    const F2 f = fadd2(y, F2{-n.x, -n.y});
    constexpr float K5 = BS_C5 * 0x1p-23f, K4 = BS_C4 * 0x1p-23f, K3 = BS_C3 * 0x1p-23f;
    constexpr float K2 = BS_C2 * 0x1p-23f, K1 = BS_C1 * 0x1p-23f, K0 = BS_C0 * 0x1p-23f;
    p = ffma2(F2{K5, K5}, f, F2{K4, K4});
    p = ffma2(p, f, F2{K3, K3});
    p = ffma2(p, f, F2{K2, K2});
    p = ffma2(p, f, F2{K1, K1});
    p = ffma2(p, f, F2{K0, K0});
}
__device__ __forceinline__ uint64_t pair_f2i(uint32_t w, float c, float nmc, float magic) {
    F2 t, p;
    pair_core(w, c, nmc, magic, t, p);
    const uint64_t m0 = f2u64_rz(__uint_as_float(add_alu(__float_as_uint(p.x), shl23_alu(__float_as_uint(t.x)))));
    const uint64_t m1 = f2u64_rz(__uint_as_float(add_alu(__float_as_uint(p.y), shl23_alu(__float_as_uint(t.y)))));
    return m0 + m1;
}
__device__ __forceinline__ void pair_split(uint32_t w, float c, float nmc, float magic, uint32_t& hi, uint32_t& lo) {
    F2 t, p;
    pair_core_s(w, c, nmc, magic, t, p);
    const F2 x{__uint_as_float(add_alu(__float_as_uint(p.x), shl23_alu(__float_as_uint(t.x)))),
               __uint_as_float(add_alu(__float_as_uint(p.y), shl23_alu(__float_as_uint(t.y))))};
    const F2 t1 = fadd2_rz(x, F2{0x1p23f, 0x1p23f});
    const F2 fl = fadd2(t1, F2{-0x1p23f, -0x1p23f});
    const F2 r = fadd2(x, F2{-fl.x, -fl.y});
    const F2 t2 = ffma2_rz(r, F2{0x1p23f, 0x1p23f}, F2{0x1p23f, 0x1p23f});
    hi += __float_as_uint(t1.x) + __float_as_uint(t1.y);
    lo += __float_as_uint(t2.x) + __float_as_uint(t2.y);
}
__device__ __forceinline__ uint32_t clamp2(uint32_t w, uint32_t L02) { return hmax2_nan_u32(w, L02); }
// 16 masses: v0 by F2I, v1 by the split floor (MODE 3); all F2I (MODE 4); all split (MODE 5)
template <int MODE>
__device__ __forceinline__ uint64_t mass16_v(uint4 v0, uint4 v1, float c, float nmc, float magic, uint32_t L02) {
    v0.x = clamp2(v0.x, L02); v0.y = clamp2(v0.y, L02); v0.z = clamp2(v0.z, L02); v0.w = clamp2(v0.w, L02);
    v1.x = clamp2(v1.x, L02); v1.y = clamp2(v1.y, L02); v1.z = clamp2(v1.z, L02); v1.w = clamp2(v1.w, L02);
    if (MODE == 4 || MODE == 7) {
        return ((pair_f2i(v0.x, c, nmc, magic) + pair_f2i(v0.y, c, nmc, magic)) +
                (pair_f2i(v0.z, c, nmc, magic) + pair_f2i(v0.w, c, nmc, magic))) +
               ((pair_f2i(v1.x, c, nmc, magic) + pair_f2i(v1.y, c, nmc, magic)) +
                (pair_f2i(v1.z, c, nmc, magic) + pair_f2i(v1.w, c, nmc, magic)));
    }
    if (MODE == 6) {
        uint32_t hi = 0, lo = 0;
        pair_split(v1.w, c, nmc, magic, hi, lo);
        pair_split(v1.z, c, nmc, magic, hi, lo);
        const uint32_t off4 = 4u * 0x4B000000u;
        return ((pair_f2i(v0.x, c, nmc, magic) + pair_f2i(v0.y, c, nmc, magic)) +
                (pair_f2i(v0.z, c, nmc, magic) + pair_f2i(v0.w, c, nmc, magic))) +
               (pair_f2i(v1.x, c, nmc, magic) + pair_f2i(v1.y, c, nmc, magic)) +
               ((uint64_t)(hi - off4) << 23) + (uint64_t)(lo - off4);
    }
    uint32_t hi = 0, lo = 0;
    pair_split(v1.x, c, nmc, magic, hi, lo);
    pair_split(v1.y, c, nmc, magic, hi, lo);
    pair_split(v1.z, c, nmc, magic, hi, lo);
    pair_split(v1.w, c, nmc, magic, hi, lo);
    if (MODE == 5) {
        pair_split(v0.x, c, nmc, magic, hi, lo);
        pair_split(v0.y, c, nmc, magic, hi, lo);
        pair_split(v0.z, c, nmc, magic, hi, lo);
        pair_split(v0.w, c, nmc, magic, hi, lo);
        const uint32_t off16 = 16u * 0x4B000000u;
        return ((uint64_t)(hi - off16) << 23) + (uint64_t)(lo - off16);
    }
    const uint32_t off8 = 8u * 0x4B000000u;
    return ((pair_f2i(v0.x, c, nmc, magic) + pair_f2i(v0.y, c, nmc, magic)) +
            (pair_f2i(v0.z, c, nmc, magic) + pair_f2i(v0.w, c, nmc, magic))) +
           ((uint64_t)(hi - off8) << 23) + (uint64_t)(lo - off8);
}

template <int CL, int NB, int NMW, int NXW, int MINB, int MODE>
__global__ void __launch_bounds__((NMW + NXW + 2) * 32, MINB)
    skel(const uint16_t* __restrict__ bank, const int* __restrict__ rows, int nrows, int V, int SL,
         unsigned long long* outZ) {
    constexpr int D = 2 * NB;
    constexpr int NT = (NMW + NXW + 2) * 32;
    constexpr int PROD = NMW + NXW, EPI = NMW + NXW + 1;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(128) uint8_t smem[];
    auto& sh = *reinterpret_cast<Sh<CL, NB>*>(smem);
    uint16_t* bufs = reinterpret_cast<uint16_t*>(smem + ((sizeof(Sh<CL, NB>) + 127) & ~size_t(127)));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rank = (int)cluster.block_rank();
    const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;
    const int e_lo = rank * SL;
    const int len = max(0, min(SL, V - e_lo));
    const int ntile = (len + TILE - 1) / TILE;
    if (tid == 0) {
        for (int i = 0; i < NB; ++i) {
            mbar_init(&sh.full[i], 1);
            mbar_init(&sh.empty[i], NMW);
        }
        for (int i = 0; i < D; ++i) {
            mbar_init(&sh.maxbar[i], 1);
            mbar_init(&sh.sumbar[i], 1);
            mbar_init(&sh.sumready[i], NMW);
            mbar_init(&sh.eempty[i], 1);
        }
        fence_mbar_init();
    }
    cluster.sync();
    const int nmine = (nrows - cid + ncl - 1) / ncl;  // rows cid, cid + ncl, ...
    const float c = 1.4426950408889634f;
    const int S = 44;
    (void)NT;
    if (warp == PROD) {
        if (lane == 0) {
            for (int i = 0; i < nmine; ++i) {
                const int bi = i % NB;
                if (i >= NB) mbar_wait(&sh.empty[bi], ((i / NB) - 1) & 1);
                const uint16_t* src = bank + (size_t)rows[cid + i * ncl] * V + e_lo;
                uint16_t* buf = bufs + (size_t)bi * SL;
                const int nb = len & ~7;
                mbar_arrive_expect_tx(&sh.full[bi], (uint32_t)nb * 2u);
                bulk_g2s(buf, src, (uint32_t)nb * 2u, &sh.full[bi], policy_evict_first());
            }
        }
    } else if (warp == EPI) {
        for (int i = 0; i < nmine; ++i) {
            const int s = i % D;
            {
                mbar_wait(&sh.sumready[s], (i / D) & 1);
                unsigned long long cs = 0;
                for (int w = 0; w < NMW; ++w) cs += sh.wsum[s][w];
                if (lane == 0) mbar_arrive_expect_tx(&sh.sumbar[s], (uint32_t)(CL * 16));
                __syncwarp();
                if (lane < CL) st_async_v4(&sh.csum[s][rank], make_uint4((uint32_t)cs, (uint32_t)(cs >> 32), 0u, 0u),
                                           &sh.sumbar[s], (uint32_t)lane);
                mbar_wait_cluster(&sh.sumbar[s], (i / D) & 1);
                unsigned long long Z = 0;
                for (int r = 0; r < CL; ++r) Z += (uint64_t)sh.csum[s][r].x | ((uint64_t)sh.csum[s][r].y << 32);
                if (rank == 0 && lane == 0) outZ[cid + i * ncl] = Z;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh.eempty[s]);
        }
    } else if (warp >= NMW) {  // max warps
        const int xw = warp - NMW;
        for (int i = 0; i < nmine; ++i) {
            const int s = i % D, bi = i % NB;
            if (i >= D) mbar_wait(&sh.eempty[s], ((i / D) - 1) & 1);
            mbar_wait(&sh.full[bi], (i / NB) & 1);
            const uint16_t* buf = bufs + (size_t)bi * SL;
            uint32_t mx = 0xFF80FF80u, mx1 = 0xFF80FF80u;
            const int nfull = len / TILE;
            int t = xw;
            if (MODE != 2) {
                for (; t + 3 * NXW < nfull; t += 4 * NXW) {
                    uint4 v[8];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        v[2 * u] = lds128(buf + (t + u * NXW) * TILE + lane * 8);
                        v[2 * u + 1] = lds128(buf + (t + u * NXW) * TILE + TILE / 2 + lane * 8);
                    }
#pragma unroll
                    for (int u = 0; u < 8; u += 2) {
                        mx = hmax2_nan_u32(mx, hmax2_nan_u32(hmax2_nan_u32(v[u].x, v[u].y), hmax2_nan_u32(v[u].z, v[u].w)));
                        mx1 = hmax2_nan_u32(mx1, hmax2_nan_u32(hmax2_nan_u32(v[u + 1].x, v[u + 1].y),
                                                               hmax2_nan_u32(v[u + 1].z, v[u + 1].w)));
                    }
                }
                for (; t < nfull; t += NXW) {
                    const uint4 v0 = lds128(buf + t * TILE + lane * 8);
                    const uint4 v1 = lds128(buf + t * TILE + TILE / 2 + lane * 8);
                    mx = hmax2_nan_u32(mx, hmax2_nan_u32(hmax2_nan_u32(v0.x, v0.y), hmax2_nan_u32(v0.z, v0.w)));
                    mx1 = hmax2_nan_u32(mx1, hmax2_nan_u32(hmax2_nan_u32(v1.x, v1.y), hmax2_nan_u32(v1.z, v1.w)));
                }
            }
            mx = hmax2_nan_u32(mx, mx1);
            float fm = fmaxf(bf16lo(mx), bf16hi(mx));
#pragma unroll
            for (int k2 = 16; k2; k2 >>= 1) fm = fmaxf(fm, __shfl_xor_sync(0xFFFFFFFFu, fm, k2));
            if (NXW > 1) {
                if (lane == 0) sh.wmax[xw] = fm;
                named_bar(2, NXW * 32);
                for (int w = 0; w < NXW; ++w) fm = fmaxf(fm, sh.wmax[w]);
            }
            if (xw == 0) {
                if (lane == 0) mbar_arrive_expect_tx(&sh.maxbar[s], (uint32_t)(CL * 16));
                __syncwarp();
                if (lane < CL) st_async_v4(&sh.cmax[s][rank], make_uint4(__float_as_uint(fm), 0u, 0u, 0u),
                                           &sh.maxbar[s], (uint32_t)lane);
            }
            if (NXW > 1) named_bar(2, NXW * 32);
        }
    } else {  // mass warps
        MassParams mp;
        mp.c = c;
        mp.clampv = -(float)(S + 2);
        mp.magic = 12582912.0f + (float)S;
        for (int i = 0; i < nmine; ++i) {
            const int s = i % D, bi = i % NB;
            mbar_wait_cluster(&sh.maxbar[s], (i / D) & 1);
            float m = -INFINITY;
#pragma unroll
            for (int r = 0; r < CL; ++r) m = fmaxf(m, __uint_as_float(sh.cmax[s][r].x));
            mbar_wait(&sh.full[bi], (i / NB) & 1);
            const uint16_t* buf = bufs + (size_t)bi * SL;
            uint64_t wacc = 0;
            if (MODE >= 3) {
                const float nmc = -__fmul_rn(m, c);
                // bf16 clamp L0 with y(L0) ~ -(S + 10): elements below have mass 0 either way
                const float l0f = (-nmc - (float)(S + 10)) / c;
                const uint32_t L0 = __float_as_uint(l0f) >> 16;
                const uint32_t L02 = L0 | (L0 << 16);
                const float magic = 12582912.0f + (float)S;
                const int nfull = len / TILE;
                for (int t = warp; t < nfull; t += NMW) {
                    const int e0 = t * TILE + lane * 8;
                    const uint64_t acc = mass16_v<MODE>(lds128(buf + e0), lds128(buf + e0 + TILE / 2), c, nmc, magic, L02);
                    if (MODE == 7) wacc += acc;
                    else wacc += warp_sum_u51(acc);
                }
            }
            if (MODE == 0) {
                mp.nmc = -__fmul_rn(m, c);
                const int nfull = len / TILE;
                for (int t = warp; t < nfull; t += NMW) {
                    const int e0 = t * TILE + lane * 8;
                    const uint64_t acc = mass16_mixed(lds128(buf + e0), lds128(buf + e0 + TILE / 2), mp);
                    wacc += warp_sum_u51(acc);
                }
            }
            if (lane == 0) sh.wsum[s][warp] = wacc;
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sh.sumready[s]);
                mbar_arrive(&sh.empty[bi]);
            }
        }
    }
    cluster.sync();
}

template <int CL, int NB, int NMW, int NXW, int MINB, int MODE>
void run(const char* name, const uint16_t* bank, const int* rows, int nrows, int V, unsigned long long* outZ,
         int nsm) {
    auto k = skel<CL, NB, NMW, NXW, MINB, MODE>;
    const int SL = ((V + CL - 1) / CL + 7) / 8 * 8;
    const size_t smem = ((sizeof(Sh<CL, NB>) + 127) & ~size_t(127)) + (size_t)NB * SL * 2;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        printf("%-28s smem %zu: %s\n", name, smem, cudaGetErrorString(e));
        cudaGetLastError();
        return;
    }
    if (CL > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL * nsm);
    cfg.blockDim = dim3((NMW + NXW + 2) * 32);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    if (e != cudaSuccess || ncl == 0) {
        printf("%-28s occupancy: %s (%d)\n", name, cudaGetErrorString(e), ncl);
        cudaGetLastError();
        return;
    }
    cfg.gridDim = dim3(CL * ncl);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, k, (const uint16_t*)bank, rows, nrows, V, SL, outZ);
    cudaEventRecord(a);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) cudaLaunchKernelEx(&cfg, k, (const uint16_t*)bank, rows, nrows, V, SL, outZ);
    cudaEventRecord(b);
    e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const double gbs = (double)nrows * V * 2 / (ms * 1e-3) / 1e9;
    printf("%-28s clusters %3d (SMs ~%3d) smem %6zu: %8.1f us  %6.0f GB/s  %6.2f rows/us  %s\n", name, ncl,
           ncl * CL / MINB, smem, ms * 1e3, gbs, nrows / (ms * 1e3), cudaGetErrorString(e));
}

int main() {
    const int V = 151936, nbank = 8192, nrows = 4096;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint16_t* bank;
    cudaMalloc(&bank, (size_t)nbank * V * 2);
    // random bf16 noise in [-4, 4)
    std::vector<uint16_t> h(V);
    for (int i = 0; i < V; ++i) {
        float f = ((rand() & 0xFFFF) / 65536.0f) * 8.f - 4.f;
        uint32_t u;
        memcpy(&u, &f, 4);
        h[i] = (uint16_t)(u >> 16);
    }
    for (int r = 0; r < nbank; ++r) cudaMemcpy(bank + (size_t)r * V, h.data(), (size_t)V * 2, cudaMemcpyHostToDevice);
    std::vector<int> hr(nrows);
    for (int i = 0; i < nrows; ++i) hr[i] = rand() % nbank;
    int* rows;
    cudaMalloc(&rows, nrows * 4);
    cudaMemcpy(rows, hr.data(), nrows * 4, cudaMemcpyHostToDevice);
    unsigned long long* outZ;
    cudaMalloc(&outZ, nrows * 8);
    printf("V=%d rows=%d (%.0f MB), %d SMs\n", V, nrows, (double)nrows * V * 2 / 1e6, nsm);
    // MODE 0 full; 1 max only; 2 copy only; 3 mixed ALU-unpack; 4 all F2I; 5 all split; 6 3/4 F2I; 7 m4 no REDUX
    run<4, 3, 16, 2, 1, 4>("cl4 nb3 mw16 1/SM m4", bank, rows, nrows, V, outZ, nsm);
    run<4, 3, 16, 2, 1, 6>("cl4 nb3 mw16 1/SM m6", bank, rows, nrows, V, outZ, nsm);
    run<4, 3, 16, 2, 1, 7>("cl4 nb3 mw16 1/SM m7", bank, rows, nrows, V, outZ, nsm);
    run<4, 3, 20, 2, 1, 4>("cl4 nb3 mw20 1/SM m4", bank, rows, nrows, V, outZ, nsm);
    run<4, 3, 20, 2, 1, 6>("cl4 nb3 mw20 1/SM m6", bank, rows, nrows, V, outZ, nsm);
    run<4, 3, 12, 2, 1, 4>("cl4 nb3 mw12 1/SM m4", bank, rows, nrows, V, outZ, nsm);
    run<4, 3, 16, 1, 1, 4>("cl4 nb3 mw16 x1 1/SM m4", bank, rows, nrows, V, outZ, nsm);
    run<4, 3, 16, 4, 1, 4>("cl4 nb3 mw16 x4 1/SM m4", bank, rows, nrows, V, outZ, nsm);
    run<8, 2, 8, 2, 2, 4>("cl8 nb2 mw8 2/SM m4", bank, rows, nrows, V, outZ, nsm);
    run<8, 2, 8, 2, 2, 6>("cl8 nb2 mw8 2/SM m6", bank, rows, nrows, V, outZ, nsm);
    run<8, 5, 20, 2, 1, 4>("cl8 nb5 mw20 1/SM m4", bank, rows, nrows, V, outZ, nsm);
    cudaDeviceSynchronize();
    printf("done: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
