// Standalone timing of the cluster kernel's per-slice mass loop (verify_cluster.cuh, mass
// warps): one CTA per SM, 8 warps, a 19,456-element bf16 slice in shared memory, tiles of
// 512 elements round-robin over the warps, per-tile exact warp sums.  Reports cycles per
// slice for the variants: mixed conversion (F2I + FMA-pipe split), F2I only, split only,
// and 1 vs 2 CTAs per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2605_08862_b200/csrc -o /tmp/ubml scripts/ubench_massloop.cu
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "verify_math.cuh"

using namespace bs;
constexpr int SL = 19456, TILE = 512, NT = SL / TILE, NW = 8;

// scalar form, every constant a compile-time immediate (S = 44, T = 1): FFMA/FADD imm-forms
__device__ __forceinline__ uint64_t mass1_imm(float l, float nmc) {
    constexpr float c = 1.4426950408889634f;
    float y = __fmaf_rn(l, c, nmc);
    y = fmaxf(y, -46.f);
    const float t = __fadd_rn(y, 12582912.0f + 44.f);
    const float n = __fadd_rn(t, -(12582912.0f + 44.f));
    const float f = __fsub_rn(y, n);
    float p = __fmaf_rn(BS_C5, f, BS_C4);
    p = __fmaf_rn(p, f, BS_C3);
    p = __fmaf_rn(p, f, BS_C2);
    p = __fmaf_rn(p, f, BS_C1);
    p = __fmaf_rn(p, f, BS_C0);
    return f2u64_rz(__uint_as_float(__float_as_uint(p) + (__float_as_uint(t) << 23)));
}
__device__ __forceinline__ uint64_t mass16_imm(const uint4 v0, const uint4 v1, float nmc) {
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint64_t a = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) a += mass1_imm(bf16lo(w[i]), nmc) + mass1_imm(bf16hi(w[i]), nmc);
    return a;
}
// scalar imm-form polynomial + split floor (no F2I), raw-bit sums
__device__ __forceinline__ void split1_imm(float l, float nmc, uint32_t& hi, uint32_t& lo) {
    constexpr float c = 1.4426950408889634f;
    float y = __fmaf_rn(l, c, nmc);
    y = fmaxf(y, -46.f);
    const float t = __fadd_rn(y, 12582912.0f + 44.f);
    const float n = __fadd_rn(t, -(12582912.0f + 44.f));
    const float f = __fsub_rn(y, n);
    float p = __fmaf_rn(BS_C5 * 0x1p-23f, f, BS_C4 * 0x1p-23f);
    p = __fmaf_rn(p, f, BS_C3 * 0x1p-23f);
    p = __fmaf_rn(p, f, BS_C2 * 0x1p-23f);
    p = __fmaf_rn(p, f, BS_C1 * 0x1p-23f);
    p = __fmaf_rn(p, f, BS_C0 * 0x1p-23f);
    const float x = __uint_as_float(__float_as_uint(p) + (__float_as_uint(t) << 23));
    const float t1 = __fadd_rz(x, 0x1p23f);
    const float r = __fsub_rn(x, __fadd_rn(t1, -0x1p23f));
    const float t2 = __fmaf_rz(r, 0x1p23f, 0x1p23f);
    hi += __float_as_uint(t1);
    lo += __float_as_uint(t2);
}
__device__ __forceinline__ uint64_t mass16_split_imm(const uint4 v0, const uint4 v1, float nmc) {
    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint32_t hi = 0, lo = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        split1_imm(bf16lo(w[i]), nmc, hi, lo);
        split1_imm(bf16hi(w[i]), nmc, hi, lo);
    }
    const uint32_t off16 = 16u * 0x4B000000u;
    return ((uint64_t)(hi - off16) << 23) + (uint64_t)(lo - off16);
}

template <int MODE>
__global__ void __launch_bounds__(NW * 32) massloop(const uint16_t* src, unsigned long long* out, long long* cyc,
                                                    int reps, float m) {
    __shared__ __align__(16) uint16_t buf[SL];
    __shared__ unsigned long long tsum[NT];
    for (int i = threadIdx.x; i < SL; i += blockDim.x) buf[i] = src[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    MassParams mp;
    mp.c = 1.4426950f;
    mp.nmc = -__fmul_rn(m, mp.c);
    mp.clampv = -46.f;
    mp.magic = 12582912.0f + 44.f;
    unsigned long long tot = 0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        uint64_t wacc = 0;
        for (int t = warp; t < NT; t += NW) {
            const int e0 = t * TILE + lane * 16;
            const uint4 v0 = lds128(buf + e0), v1 = lds128(buf + e0 + 8);
            uint64_t acc;
            if (MODE == 0) acc = mass16_mixed(v0, v1, mp);
            else if (MODE == 1) acc = mass8(v0, mp) + mass8(v1, mp);
            else if (MODE == 2) acc = mass16_split(v0, v1, mp);
            else if (MODE == 3) acc = mass16_imm(v0, v1, mp.nmc);
            else acc = mass16_split_imm(v0, v1, mp.nmc);
            const uint64_t ts = warp_sum_u51(acc);
            if (lane == 0) tsum[t] = ts;
            wacc += ts;
        }
        named_bar(1, NW * 32);
        tot += wacc;
    }
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * NW + warp] = tot;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint16_t h[SL];
    unsigned s = 12345;
    for (int i = 0; i < SL; ++i) {
        s = s * 1664525u + 1013904223u;
        const float v = ((int)(s >> 9) % 2000 - 1000) * 0.005f;  // [-5, 5]
        unsigned b;
        memcpy(&b, &v, 4);
        h[i] = (uint16_t)(b >> 16);
    }
    uint16_t* d;
    unsigned long long* o;
    long long* c;
    cudaMalloc(&d, sizeof h);
    cudaMalloc(&o, sizeof(unsigned long long) * 2 * sms * NW);
    cudaMalloc(&c, sizeof(long long) * 2 * sms);
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    const int reps = getenv("REPS") ? atoi(getenv("REPS")) : 50;
    const char* names[5] = {"mixed", "f2i", "split", "imm", "splimm"};
    for (int mode = 0; mode < 5; ++mode)
        for (int per = 1; per <= 2; ++per) {
            const int grid = per * sms;
            for (int w = 0; w < 2; ++w) {
                if (mode == 0) massloop<0><<<grid, NW * 32>>>(d, o, c, reps, 6.0f);
                if (mode == 1) massloop<1><<<grid, NW * 32>>>(d, o, c, reps, 6.0f);
                if (mode == 2) massloop<2><<<grid, NW * 32>>>(d, o, c, reps, 6.0f);
                if (mode == 3) massloop<3><<<grid, NW * 32>>>(d, o, c, reps, 6.0f);
                if (mode == 4) massloop<4><<<grid, NW * 32>>>(d, o, c, reps, 6.0f);
            }
            cudaDeviceSynchronize();
            long long hc[512];
            cudaMemcpy(hc, c, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < grid; ++i) avg += hc[i];
            avg /= grid;
            unsigned long long ho[8];
            cudaMemcpy(ho, o, sizeof ho, cudaMemcpyDeviceToHost);
            printf("[sum %llx] ", ho[0] + ho[1] + ho[2] + ho[3] + ho[4] + ho[5] + ho[6] + ho[7]);
            printf("%-6s %d CTA/SM: %8.0f cycles per slice (%.2f us at 1.965 GHz), %.2f el/clk/SM\n", names[mode], per,
                   avg / reps, avg / reps / 1965.0, (double)SL * per / (avg / reps));
        }
    return 0;
}
