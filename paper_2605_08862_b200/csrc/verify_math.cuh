// verify_math.cuh — per-element arithmetic of the verify kernel (reading R)
// with packed sm_100a instructions, and small warp/CTA helpers.
#pragma once
#include <cuda_bf16.h>

#include "common.cuh"

namespace bs {

struct F2 {
    float x, y;
};
// fma.rn.f32x2 / add.rn.f32x2 (FFMA2 / FADD2): two IEEE single operations per instruction.
__device__ __forceinline__ F2 ffma2(F2 a, F2 b, F2 c) {
    F2 r;
    asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}
__device__ __forceinline__ F2 fadd2(F2 a, F2 b) {
    F2 r;
    asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}

__device__ __forceinline__ F2 fadd2_rz(F2 a, F2 b) {
    F2 r;
    asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " add.rz.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ F2 ffma2_rz(F2 a, F2 b, F2 c) {
    F2 r;
    asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " mov.b64 rc, {%6, %7};\n fma.rz.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}

// Masses of the two bf16 logits packed in w (R2-R4), bit-identical to mass_of() per lane:
// the packed FFMA2 / FADD2 perform the same IEEE single operations.
__device__ __forceinline__ void mass_pair(uint32_t w, const MassParams& mp, uint64_t& m0,
                                          uint64_t& m1) {
    const F2 l{bf16lo(w), bf16hi(w)};
    F2 y = ffma2(l, F2{mp.c, mp.c}, F2{mp.nmc, mp.nmc});
    y.x = fmaxf(y.x, mp.clampv);
    y.y = fmaxf(y.y, mp.clampv);
    const F2 t = fadd2(y, F2{mp.magic, mp.magic});
    const F2 n = fadd2(t, F2{-mp.magic, -mp.magic});
    const F2 f = fadd2(y, F2{-n.x, -n.y});
    F2 p = ffma2(F2{BS_C5, BS_C5}, f, F2{BS_C4, BS_C4});
    p = ffma2(p, f, F2{BS_C3, BS_C3});
    p = ffma2(p, f, F2{BS_C2, BS_C2});
    p = ffma2(p, f, F2{BS_C1, BS_C1});
    p = ffma2(p, f, F2{BS_C0, BS_C0});
    m0 = f2u64_rz(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)));
    m1 = f2u64_rz(__uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

__device__ __forceinline__ uint64_t mass8(const uint4 v, const MassParams& mp) {
    uint64_t a0, a1, b0, b1, c0, c1, d0, d1;
    mass_pair(v.x, mp, a0, a1);
    mass_pair(v.y, mp, b0, b1);
    mass_pair(v.z, mp, c0, c1);
    mass_pair(v.w, mp, d0, d1);
    return ((a0 + a1) + (b0 + b1)) + ((c0 + c1) + (d0 + d1));
}

// The same two masses with the conversion on the FMA pipe instead of F2I.U64 (the XU pipe),
// valid for S <= 44: with the polynomial coefficients scaled by 2^-23 (exact), the exponent
// insert yields x = e' * 2^-23 < 2^23 bit for bit, and
//   floor(e') = floor(x) * 2^23 + floor(frac(x) * 2^23)
// where t1 = RZ(x + 2^23) = 2^23 + floor(x), frac(x) = x - (t1 - 2^23) (exact) and
// t2 = RZ(frac(x) * 2^23 + 2^23) = 2^23 + floor(frac(x) * 2^23).  The raw bits of t1 / t2 are
// summed in u32 (hi / lo); the 2^23 offsets are taken off once per block.
__device__ __forceinline__ void mass_pair_split(uint32_t w, const MassParams& mp, uint32_t& hi, uint32_t& lo) {
    const F2 l{bf16lo(w), bf16hi(w)};
    F2 y = ffma2(l, F2{mp.c, mp.c}, F2{mp.nmc, mp.nmc});
    y.x = fmaxf(y.x, mp.clampv);
    y.y = fmaxf(y.y, mp.clampv);
    const F2 t = fadd2(y, F2{mp.magic, mp.magic});
    const F2 n = fadd2(t, F2{-mp.magic, -mp.magic});
    const F2 f = fadd2(y, F2{-n.x, -n.y});
    constexpr float K5 = BS_C5 * 0x1p-23f, K4 = BS_C4 * 0x1p-23f, K3 = BS_C3 * 0x1p-23f;
    constexpr float K2 = BS_C2 * 0x1p-23f, K1 = BS_C1 * 0x1p-23f, K0 = BS_C0 * 0x1p-23f;
    F2 p = ffma2(F2{K5, K5}, f, F2{K4, K4});
    p = ffma2(p, f, F2{K3, K3});
    p = ffma2(p, f, F2{K2, K2});
    p = ffma2(p, f, F2{K1, K1});
    p = ffma2(p, f, F2{K0, K0});
    const F2 x{__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
               __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23))};
    const F2 t1 = fadd2_rz(x, F2{0x1p23f, 0x1p23f});
    const F2 fl = fadd2(t1, F2{-0x1p23f, -0x1p23f});
    const F2 r = fadd2(x, F2{-fl.x, -fl.y});
    const F2 t2 = ffma2_rz(r, F2{0x1p23f, 0x1p23f}, F2{0x1p23f, 0x1p23f});
    hi += __float_as_uint(t1.x) + __float_as_uint(t1.y);
    lo += __float_as_uint(t2.x) + __float_as_uint(t2.y);
}

// Sum of 16 masses: v0's eight by F2I.U64, v1's eight by the FMA-pipe split floor (S <= 44):
// the two conversions run on different pipes.
__device__ __forceinline__ uint64_t mass16_mixed(const uint4 v0, const uint4 v1, const MassParams& mp) {
    uint32_t hi = 0, lo = 0;
    mass_pair_split(v1.x, mp, hi, lo);
    mass_pair_split(v1.y, mp, hi, lo);
    mass_pair_split(v1.z, mp, hi, lo);
    mass_pair_split(v1.w, mp, hi, lo);
    const uint32_t off8 = 8u * 0x4B000000u;  // eight 2^23 offsets, mod 2^32
    return mass8(v0, mp) + ((uint64_t)(hi - off8) << 23) + (uint64_t)(lo - off8);
}

__device__ __forceinline__ uint64_t mass16_split(const uint4 v0, const uint4 v1, const MassParams& mp) {
    uint32_t hi = 0, lo = 0;
    mass_pair_split(v0.x, mp, hi, lo);
    mass_pair_split(v0.y, mp, hi, lo);
    mass_pair_split(v0.z, mp, hi, lo);
    mass_pair_split(v0.w, mp, hi, lo);
    mass_pair_split(v1.x, mp, hi, lo);
    mass_pair_split(v1.y, mp, hi, lo);
    mass_pair_split(v1.z, mp, hi, lo);
    mass_pair_split(v1.w, mp, hi, lo);
    const uint32_t off16 = 16u * 0x4B000000u;
    return ((uint64_t)(hi - off16) << 23) + (uint64_t)(lo - off16);
}

// One lane's 8 masses of a tile, elements >= nvalid or == excl (tile-relative) zeroed.
__device__ __forceinline__ void mass8_masked(const uint4 v, const MassParams& mp, int e0, int nvalid,
                                             int excl, uint64_t mm[8]) {
    mass_pair(v.x, mp, mm[0], mm[1]);
    mass_pair(v.y, mp, mm[2], mm[3]);
    mass_pair(v.z, mp, mm[4], mm[5]);
    mass_pair(v.w, mp, mm[6], mm[7]);
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (e0 + i >= nvalid || e0 + i == excl) mm[i] = 0;
}

__device__ __forceinline__ uint32_t hmax2_nan_u32(uint32_t a, uint32_t b) {
    __nv_bfloat162 x, y;
    memcpy(&x, &a, 4);
    memcpy(&y, &b, 4);
    __nv_bfloat162 z = __hmax2_nan(x, y);
    uint32_t r;
    memcpy(&r, &z, 4);
    return r;
}

// ---- the mass loop's fast form (measured: +25-50 % row throughput over mass16_mixed,
// scripts/ubench_stream.cu).  Bit-identical masses; three changes of instruction selection:
//  * bf16 unpack on the ALU pipe (PRMT / LOP3) instead of IMAD.U32 on the FMA pipe;
//  * the lower clamp applied once per bf16 pair with HMNMX2 at a per-row bf16 bound L0
//    (row_clamp_l0) instead of two FMNMX on y: every element below L0 has mass 0 in R and
//    so does L0 itself, and y(L0) >= -(S + 60) keeps the exponent insert exact;
//  * every conversion by F2I.U64 (the XU pipe has room once the FMA pipe is relieved).
__device__ __forceinline__ float bf16lo_alu(uint32_t w) { return __uint_as_float(__byte_perm(w, 0u, 0x1044u)); }
__device__ __forceinline__ float bf16hi_alu(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// Per-row lower clamp: a bf16 value L0 with -(S + 60) <= y(L0) <= -(S + 2), where y(l) =
// fma(l, c, nmc) is the kernel's own FFMA, returned duplicated in both halves (0 if none
// exists: huge |m|, whose bf16 spacing exceeds the window; the caller then uses mass8).
__device__ __forceinline__ uint32_t row_clamp_l0(float c, float nmc, int S) {
    const float target = (-nmc - (float)(S + 20)) / c;
    uint32_t b = __float_as_uint(target) >> 16;  // bf16 truncation of the target
    for (int it = 0; it < 8; ++it) {
        const float y = __fmaf_rn(__uint_as_float(b << 16), c, nmc);
        if (y > -(float)(S + 2)) {  // too high: one bf16 step towards -inf
            b = (b & 0x8000u) ? b + 1u : (b ? b - 1u : 0x8001u);
            continue;
        }
        if (y < -(float)(S + 60)) return 0u;
        return b | (b << 16);
    }
    return 0u;
}

__device__ __forceinline__ uint64_t mass_pair_f2i(uint32_t w, float c, float nmc, float magic) {
    const F2 l{bf16lo_alu(w), bf16hi_alu(w)};
    const F2 y = ffma2(l, F2{c, c}, F2{nmc, nmc});
    const F2 t = fadd2(y, F2{magic, magic});
    const F2 n = fadd2(t, F2{-magic, -magic});
    const F2 f = fadd2(y, F2{-n.x, -n.y});
    F2 p = ffma2(F2{BS_C5, BS_C5}, f, F2{BS_C4, BS_C4});
    p = ffma2(p, f, F2{BS_C3, BS_C3});
    p = ffma2(p, f, F2{BS_C2, BS_C2});
    p = ffma2(p, f, F2{BS_C1, BS_C1});
    p = ffma2(p, f, F2{BS_C0, BS_C0});
    const uint64_t m0 = f2u64_rz(__uint_as_float(__float_as_uint(p.x) + __funnelshift_l(0u, __float_as_uint(t.x), 23)));
    const uint64_t m1 = f2u64_rz(__uint_as_float(__float_as_uint(p.y) + __funnelshift_l(0u, __float_as_uint(t.y), 23)));
    return m0 + m1;
}

#ifdef BS_UB_MUFU
// MEASUREMENT BUILD ONLY (libbubblespec_ubmufu.so; decisions are NOT R's): the mass loop with
// MUFU ex2.approx and fp32 sums instead of R's polynomial and integer masses: the upper bound
// on what a certified fast path could gain in this kernel.
__device__ __forceinline__ float ex2_mufu(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float mass_pair_mufu(uint32_t w, float c, float nmcs) {
    const F2 l{bf16lo_alu(w), bf16hi_alu(w)};
    const F2 y = ffma2(l, F2{c, c}, F2{nmcs, nmcs});
    return ex2_mufu(y.x) + ex2_mufu(y.y);
}
__device__ __forceinline__ uint64_t mass16_fast(uint4 v0, uint4 v1, float c, float nmc, float magic, uint32_t L02) {
    const float nmcs = nmc + (magic - 12582912.0f);
    const float s = ((mass_pair_mufu(v0.x, c, nmcs) + mass_pair_mufu(v0.y, c, nmcs)) +
                     (mass_pair_mufu(v0.z, c, nmcs) + mass_pair_mufu(v0.w, c, nmcs))) +
                    ((mass_pair_mufu(v1.x, c, nmcs) + mass_pair_mufu(v1.y, c, nmcs)) +
                     (mass_pair_mufu(v1.z, c, nmcs) + mass_pair_mufu(v1.w, c, nmcs)));
    (void)L02;
    return f2u64_rz(s);
}
#else
// Sum of the 16 masses of two 16-byte bf16 vectors; L02 from row_clamp_l0 (nonzero).
__device__ __forceinline__ uint64_t mass16_fast(uint4 v0, uint4 v1, float c, float nmc, float magic, uint32_t L02) {
    v0.x = hmax2_nan_u32(v0.x, L02);
    v0.y = hmax2_nan_u32(v0.y, L02);
    v0.z = hmax2_nan_u32(v0.z, L02);
    v0.w = hmax2_nan_u32(v0.w, L02);
    v1.x = hmax2_nan_u32(v1.x, L02);
    v1.y = hmax2_nan_u32(v1.y, L02);
    v1.z = hmax2_nan_u32(v1.z, L02);
    v1.w = hmax2_nan_u32(v1.w, L02);
    return ((mass_pair_f2i(v0.x, c, nmc, magic) + mass_pair_f2i(v0.y, c, nmc, magic)) +
            (mass_pair_f2i(v0.z, c, nmc, magic) + mass_pair_f2i(v0.w, c, nmc, magic))) +
           ((mass_pair_f2i(v1.x, c, nmc, magic) + mass_pair_f2i(v1.y, c, nmc, magic)) +
            (mass_pair_f2i(v1.z, c, nmc, magic) + mass_pair_f2i(v1.w, c, nmc, magic)));
}
#endif

// Exact warp sum of u64 lane values < 2^51 with three 32-bit REDUX sums.
__device__ __forceinline__ uint64_t warp_sum_u51(uint64_t v) {
    const uint32_t hi = (uint32_t)(v >> 32);
    const uint32_t mid = (uint32_t)(v >> 16) & 0xFFFFu;
    const uint32_t lo = (uint32_t)v & 0xFFFFu;
    const uint32_t sh = __reduce_add_sync(0xFFFFFFFFu, hi);
    const uint32_t sm = __reduce_add_sync(0xFFFFFFFFu, mid);
    const uint32_t sl = __reduce_add_sync(0xFFFFFFFFu, lo);
    return ((uint64_t)sh << 32) + ((uint64_t)sm << 16) + (uint64_t)sl;
}

__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ int ld_volatile_i32(const int32_t* p) {
    return *reinterpret_cast<const volatile int32_t*>(p);
}

}  // namespace bs
