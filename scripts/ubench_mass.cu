// Microbenchmark of the per-element mass arithmetic (reading R) on sm_100a, no memory
// traffic: elements / clock / SM for (A) F2I.U64 conversion, (B) integer mantissa shift,
// (C) a 50/50 mix, and (D) the exp polynomial alone.  Also checks A == B bit for bit.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_mass ubench_mass.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct F2 { float x, y; };
__device__ __forceinline__ F2 ffma2(F2 a, F2 b, F2 c) {
    F2 r;
    asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}
__device__ __forceinline__ F2 fadd2(F2 a, F2 b) {
    F2 r;
    asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}
__device__ __forceinline__ unsigned long long f2u(float x) {
    unsigned long long r;
    asm("cvt.rzi.u64.f32 %0, %1;" : "=l"(r) : "f"(x));
    return r;
}
#define C0 0x1.000002p+0f
#define C1 0x1.62e428p-1f
#define C2 0x1.ebf918p-3f
#define C3 0x1.c6b6e4p-5f
#define C4 0x1.3d0c54p-7f
#define C5 0x1.5c08e6p-10f

// p, t -> mass: (A) exponent insert + F2I; (B) integer: M = mantissa|hidden, shift by
// k = exp(p) + (bits(t) - bits(1.5*2^23)) - 150 ... as a 64-bit funnel right shift.
template <int MODE>
__device__ __forceinline__ void pair(uint32_t w, float c, float nmc, float clampv, float magic,
                                     unsigned long long& m0, unsigned long long& m1) {
    F2 l{__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u)};
    F2 y = ffma2(l, F2{c, c}, F2{nmc, nmc});
    y.x = fmaxf(y.x, clampv);
    y.y = fmaxf(y.y, clampv);
    const F2 t = fadd2(y, F2{magic, magic});
    const F2 n = fadd2(t, F2{-magic, -magic});
    const F2 f = fadd2(y, F2{-n.x, -n.y});
    F2 p = ffma2(F2{C5, C5}, f, F2{C4, C4});
    p = ffma2(p, f, F2{C3, C3});
    p = ffma2(p, f, F2{C2, C2});
    p = ffma2(p, f, F2{C1, C1});
    p = ffma2(p, f, F2{C0, C0});
    if (MODE == 3) {
        m0 = __float_as_uint(p.x);
        m1 = __float_as_uint(p.y);
        return;
    }
    if (MODE == 7) {
        // mixed pipes: lane x by F2I.U64, lane y by the FP64 DADD.RZ floor (t from magic+896:
        // the x lane's exponent insert subtracts the extra 896 << 23)
        m0 = f2u(__uint_as_float(__float_as_uint(p.x) + ((__float_as_uint(t.x) - 896u) << 23)));
        const uint32_t hy = (__float_as_uint(p.y) >> 3) + (__float_as_uint(t.y) << 20);
        const double dy = __hiloint2double((int)hy, (int)(__float_as_uint(p.y) << 29));
        m1 = (unsigned long long)__double_as_longlong(__dadd_rz(dy, 4503599627370496.0)) - 0x4330000000000000ull;
        return;
    }
    if (MODE == 6) {
        // FP64 floor: double(e') from the float bits (re-bias +896 folded into the shift of
        // t's bits: t's low bits are n+S+896 when magic carries +896), then
        // DADD.RZ(x, 2^52) leaves floor(x) in the low mantissa bits; the bits are summed
        // raw and count * bits(2^52) is taken off once at the end.
        const uint32_t hx = (__float_as_uint(p.x) >> 3) + (__float_as_uint(t.x) << 20);
        const uint32_t hy = (__float_as_uint(p.y) >> 3) + (__float_as_uint(t.y) << 20);
        const double dx = __hiloint2double((int)hx, (int)(__float_as_uint(p.x) << 29));
        const double dy = __hiloint2double((int)hy, (int)(__float_as_uint(p.y) << 29));
        m0 = (unsigned long long)__double_as_longlong(__dadd_rz(dx, 4503599627370496.0));
        m1 = (unsigned long long)__double_as_longlong(__dadd_rz(dy, 4503599627370496.0));
        return;
    }
    if (MODE == 4 || MODE == 5) {
        // conversion-free floor: e' = A*2^23 + B, A = floor(e'/2^23), B = floor(e' - A*2^23)
        const float e0 = __uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23));
        const float e1 = __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23));
        F2 t1;
        if (MODE == 4) {
            t1.x = __fmaf_rz(e0, 0x1p-23f, 0x1p23f);
            t1.y = __fmaf_rz(e1, 0x1p-23f, 0x1p23f);
        } else {
            uint64_t r;
            asm("{\n .reg .b64 ra, rb, rc;\n mov.b64 ra, {%1, %2};\n mov.b64 rb, {%3, %3};\n mov.b64 rc, {%4, %4};\n"
                " fma.rz.f32x2 %0, ra, rb, rc;\n}" : "=l"(r) : "f"(e0), "f"(e1), "f"(0x1p-23f), "f"(0x1p23f));
            t1.x = __uint_as_float((uint32_t)r); t1.y = __uint_as_float((uint32_t)(r >> 32));
        }
        const F2 hf = fadd2(t1, F2{-0x1p23f, -0x1p23f});
        const F2 rr = ffma2(F2{-hf.x, -hf.y}, F2{0x1p23f, 0x1p23f}, F2{e0, e1});
        F2 t2;
        t2.x = __fadd_rz(rr.x, 0x1p23f);
        t2.y = __fadd_rz(rr.y, 0x1p23f);
        const uint32_t A0 = __float_as_uint(t1.x) - 0x4B000000u, A1 = __float_as_uint(t1.y) - 0x4B000000u;
        const uint32_t B0 = __float_as_uint(t2.x) - 0x4B000000u, B1 = __float_as_uint(t2.y) - 0x4B000000u;
        m0 = ((unsigned long long)A0 << 23) + B0;
        m1 = ((unsigned long long)A1 << 23) + B1;
        return;
    }
    auto conv = [&](float pp, float tt) -> unsigned long long {
        if (MODE == 0) {
            return f2u(__uint_as_float(__float_as_uint(pp) + (__float_as_uint(tt) << 23)));
        }
        // e' = p * 2^(n+S): bits(e') = bits(p) + (S+n)<<23, value = M * 2^(E - 150)
        const uint32_t eb = __float_as_uint(pp) + (__float_as_uint(tt) << 23);
        const uint32_t M = (eb & 0x7FFFFFu) | 0x800000u;
        const int E = (int)(eb >> 23);
        // mass = M * 2^(E-150) truncated; X = M << 40 (as hi:lo), shift right by 190 - E
        const uint32_t hi = M << 8;  // X = hi * 2^32
        const int sh = 190 - E;      // >= 0 in range
        unsigned long long X = (unsigned long long)hi << 32;
        return sh >= 64 ? 0ull : (X >> sh);
    };
    if (MODE == 2) {
        m0 = conv(p.x, t.x);
        const uint32_t eb = __float_as_uint(p.y) + (__float_as_uint(t.y) << 23);
        m1 = f2u(__uint_as_float(eb));
    } else {
        m0 = conv(p.x, t.x);
        m1 = conv(p.y, t.y);
    }
}

template <int MODE>
__global__ void __launch_bounds__(512) k(const uint32_t* in, unsigned long long* out, int iters,
                                          float c, float nmc, float clampv, float magic) {
    uint32_t w[8];
    for (int i = 0; i < 8; ++i) w[i] = in[(threadIdx.x * 8 + i) & 1023];
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            unsigned long long a0, a1;
            pair<MODE>(w[i], c, nmc, clampv, magic, a0, a1);
            acc += a0 + a1;
            w[i] = w[i] * 1664525u + 1013904223u;  // next input (cheap LCG)
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void check(unsigned long long* bad) {
    __shared__ unsigned long long nb;
    if (threadIdx.x == 0) nb = 0;
    __syncthreads();
    unsigned long long local = 0, local6 = 0, local7 = 0;
    for (int r = 0; r < 64; ++r) {
        const uint32_t gid = (blockIdx.x * blockDim.x + threadIdx.x) * 64 + r;
        // y spans [-46, 1]: logits l = bf16 from hash, c and m chosen per block
        uint32_t h = gid * 2654435761u;
        h ^= h >> 15;
        const uint32_t w = (h & 0x7FFF7FFFu) ^ 0xC0000000u;  // two finite bf16 values
        const float c = 1.0f + (blockIdx.x & 15) * 0.173f;
        const float mc = 20.0f * c;
        unsigned long long a0, a1, b0, b1;
        pair<0>(w, c, -mc, -46.f, 12582912.f + 44.f, a0, a1);
        pair<4>(w, c, -mc, -46.f, 12582912.f + 44.f, b0, b1);
        local += (a0 != b0) + (a1 != b1);
        pair<5>(w, c, -mc, -46.f, 12582912.f + 44.f, b0, b1);
        local += (a0 != b0) + (a1 != b1);
        pair<6>(w, c, -mc, -46.f, 12582912.f + 44.f + 896.f, b0, b1);
        local6 += (a0 != b0 - 0x4330000000000000ull) + (a1 != b1 - 0x4330000000000000ull);
        pair<7>(w, c, -mc, -46.f, 12582912.f + 44.f + 896.f, b0, b1);
        local7 += (a0 != b0) + (a1 != b1);
    }
    atomicAdd(&nb, local);
    atomicAdd(&bad[1], local6);
    atomicAdd(&bad[2], local7);
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(bad, nb);
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    uint32_t* in;
    unsigned long long* out;
    cudaMalloc(&in, 1024 * 4);
    cudaMalloc(&out, (size_t)sms * 4 * 512 * 8);
    uint32_t h[1024];
    for (int i = 0; i < 1024; ++i) h[i] = 0x3F80BF80u + i * 2654435761u;  // arbitrary bf16 pairs
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    const float c = 1.4426950f, nmc = -1.4426950f * 8.0f, clampv = -46.f, magic = 12582912.f + 44.f;
    const int iters = 2000;
    const char* names[8] = {"F2I.U64", "integer shift", "50/50 mix", "poly only", "fp split rz", "fp split rz x2", "fp64 dadd.rz", "F2I + DADD mix"};
    for (int mode = 0; mode < 8; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            dim3 g(sms * 2), blk(512);
            if (mode == 0) k<0><<<g, blk>>>(in, out, iters, c, nmc, clampv, magic);
            if (mode == 1) k<1><<<g, blk>>>(in, out, iters, c, nmc, clampv, magic);
            if (mode == 2) k<2><<<g, blk>>>(in, out, iters, c, nmc, clampv, magic);
            if (mode == 3) k<3><<<g, blk>>>(in, out, iters, c, nmc, clampv, magic);
            if (mode == 4) k<4><<<g, blk>>>(in, out, iters, c, nmc, clampv, magic);
            if (mode == 5) k<5><<<g, blk>>>(in, out, iters, c, nmc, clampv, magic);
            if (mode == 6) k<6><<<g, blk>>>(in, out, iters, c, nmc, clampv, magic + 896.f);
            if (mode == 7) k<7><<<g, blk>>>(in, out, iters, c, nmc, clampv, magic + 896.f);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double elems = (double)sms * 2 * 512 * iters * 16;
            if (rep) printf("%-14s %8.3f ms  %6.2f elem/clk/SM (at %d MHz nominal)\n", names[mode], ms,
                            elems / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        }
    }
    // bit-equality of the conversion-free floor against F2I.U64 over a dense y sweep
    cudaMemset(out, 0, 24);
    check<<<4096, 256>>>(out);
    unsigned long long bad[3] = {0, 0, 0};
    cudaMemcpy(bad, out, 24, cudaMemcpyDeviceToHost);
    printf("mismatches vs F2I.U64 (of %d): fp split %llu, fp64 dadd %llu, F2I+DADD mix %llu\n",
           4096 * 256 * 64 * 2, bad[0], bad[1], bad[2]);
    return 0;
}
