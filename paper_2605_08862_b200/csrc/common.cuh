// common.cuh — device-side arithmetic of the BubbleSpec hot path (sm_100a).
//
// Restates, independently of the CPU oracle, the reference arithmetic R of
// DESIGN.md §3 (readings R0-R8).  Nothing here is shared with oracle/.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <utility>

namespace bs {

// ------------------------------------------------------------------ host: device scope
// Every C-ABI call runs on its context's device and leaves the caller's current device as it
// found it (one process may drive several GPUs, and the caller's framework keeps its own).
struct DeviceScope {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceScope(int dev) {
        err = cudaGetDevice(&prev);
        if (err != cudaSuccess) prev = -1;
        else if (prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceScope() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;
};

// ------------------------------------------------------------------ error word
constexpr uint32_t DEV_BAD_LOGIT = 0x1u, DEV_ALL_NEGINF = 0x2u, DEV_RANGE = 0x4u,
                   DEV_BAD_DRAFT = 0x8u, DEV_INDEX_KEY = 0x10u,
                   DEV_STALE = 0x20u;

// ------------------------------------------------------------------ Philox4x32-10 (R6)
struct U128 {
    uint32_t x0, x1, x2, x3;  // r128 = x0*2^96 + x1*2^64 + x2*2^32 + x3
};

__device__ __forceinline__ U128 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    return U128{c0, c1, c2, c3};
}

enum : uint32_t { PURPOSE_ACCEPT = 0u, PURPOSE_SAMPLE = 1u };

__device__ __forceinline__ U128 draw(uint64_t seed, uint64_t uid, uint32_t position,
                                     uint32_t purpose) {
    return philox4x32_10(position, purpose, (uint32_t)uid, (uint32_t)(uid >> 32), (uint32_t)seed,
                         (uint32_t)(seed >> 32));
}

// floor(r128 * Z / 2^128), exact: (A + (B >> 64)) >> 64 with A = rh*Z, B = rl*Z.
__device__ __forceinline__ uint64_t uniform_floor(U128 r, uint64_t Z) {
    const uint64_t rh = ((uint64_t)r.x0 << 32) | r.x1;
    const uint64_t rl = ((uint64_t)r.x2 << 32) | r.x3;
    const uint64_t a_lo = rh * Z, a_hi = __umul64hi(rh, Z);
    const uint64_t b_hi = __umul64hi(rl, Z);
    const uint64_t s = a_lo + b_hi;
    return a_hi + (s < a_lo ? 1ull : 0ull);
}

// ------------------------------------------------------------------ masses (R2-R4)
// exp2 polynomial coefficients (R3), fp32 hex.
#define BS_C0 0x1.000002p+0f
#define BS_C1 0x1.62e428p-1f
#define BS_C2 0x1.ebf918p-3f
#define BS_C3 0x1.c6b6e4p-5f
#define BS_C4 0x1.3d0c54p-7f
#define BS_C5 0x1.5c08e6p-10f

// Per-row constants of the mass map.
struct MassParams {
    float c;       // fl32(log2 e / T)
    float nmc;     // -fl32(m * c)
    float clampv;  // -(S + 2)
    float magic;   // 1.5 * 2^23 + S   (S even: RNE(magic + y) = magic + RNE(y))
};

__host__ __device__ inline int mass_shift(int V) {
    int lg = 0;
    while (((int64_t)1 << lg) < (int64_t)V) ++lg;
    int S = 62 - lg;
    return S - (S & 1);
}

__device__ __forceinline__ uint64_t f2u64_rz(float x) {
    uint64_t r;
    asm("cvt.rzi.u64.f32 %0, %1;" : "=l"(r) : "f"(x));
    return r;
}

// mass(l) = floor(2^S * p(f) * 2^n), y = fma(l, c, -mc) clamped at -(S+2),
// n = RNE(y), f = y - n.  Bit-identical to the oracle's definition (R3/R4):
// below -(S+2) the clamp yields p(0)*2^-2 < 1 -> 0, which is the definition's value.
__device__ __forceinline__ uint64_t mass_of(float l, const MassParams& mp) {
    float y = __fmaf_rn(l, mp.c, mp.nmc);
    y = fmaxf(y, mp.clampv);
    const float t = __fadd_rn(y, mp.magic);
    const float n = __fsub_rn(t, mp.magic);
    const float f = __fsub_rn(y, n);
    float p = BS_C5;
    p = __fmaf_rn(p, f, BS_C4);
    p = __fmaf_rn(p, f, BS_C3);
    p = __fmaf_rn(p, f, BS_C2);
    p = __fmaf_rn(p, f, BS_C1);
    p = __fmaf_rn(p, f, BS_C0);
    // bits(t) = bits(1.5*2^23) + S + n and (bits(1.5*2^23) << 23) == 0 mod 2^32,
    // so (bits(t) << 23) adds (S + n) to p's exponent field: e' = p * 2^(n+S).
    const uint32_t eb = __float_as_uint(p) + (__float_as_uint(t) << 23);
    return f2u64_rz(__uint_as_float(eb));
}

// Two masses at once with packed f32x2 arithmetic (FFMA2 / FADD2 on sm_100a).
// Same per-element IEEE operations as mass_of, so bit-identical.
__device__ __forceinline__ void mass_of2(float l0, float l1, const MassParams& mp, uint64_t& m0,
                                         uint64_t& m1) {
    m0 = mass_of(l0, mp);
    m1 = mass_of(l1, mp);
}

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

// ------------------------------------------------------------------ hashing (index keys)
constexpr uint64_t HASH_B = 0x9E3779B97F4A7C15ull;  // odd base of the window hash

__host__ __device__ inline uint64_t fmix64(uint64_t k) {
    k ^= k >> 33;
    k *= 0xFF51AFD7ED558CCDull;
    k ^= k >> 33;
    k *= 0xC4CEB9FE1A85EC53ull;
    k ^= k >> 33;
    return k;
}

// Table key of window w (length len, hash H) in prompt P's pool.  Never 0 (0 = empty).
__host__ __device__ inline uint64_t window_key(uint64_t H, int32_t P, int32_t len) {
    uint64_t k = fmix64(H + (uint64_t)(uint32_t)P * 0xD6E8FEB86659FD93ull +
                        (uint64_t)(uint32_t)len * 0xA0761D6478BD642Full);
    return k ? k : 1ull;
}

// Index entry: 16 bytes.
struct __align__(16) IndexEntry {
    unsigned long long key;  // 0 = empty
    uint32_t occ;            // pool position: start of an occurrence of window + path
    uint32_t meta;           // q (bits 0-7) | unique (bit 8) | cont (bit 9)
};
constexpr uint32_t META_UNIQUE = 0x100u, META_CONT = 0x200u;

// ------------------------------------------------------------------ synthetic workload
__host__ __device__ inline uint32_t h32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x;
}

// ---- programmatic dependent launch (decode-loop kernels).  Every kernel of the decode loop
// is launched with programmatic stream serialization: its CTAs may be scheduled while the
// previous kernel still runs, and pdl_wait() (griddepcontrol.wait) blocks until that kernel
// has completed and its memory is visible.  pdl_trigger() lets the next kernel launch early.
// Kernels call pdl_wait() before touching global memory, with one exception: the cluster
// verify kernel plans (reads slots, drafts, positions, lengths; writes its scheduler state)
// before its wait, which is safe because every kernel of ours that writes those inputs or
// that state (lookup, commit, every verify kernel) triggers its dependents only at exit
// (lookup: after its stores), and the kernel in between (the model / target rows) waits for
// them; user kernels launched without PDL complete before the next launch starts anyway.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_ex(bool cooperative, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    // cooperative: the launch fails instead of running when the grid cannot be co-resident
    // (the persistent verify scheduler spins on work of CTAs that would otherwise never run)
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = cooperative ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    return launch_pdl_ex(false, kernel, grid, block, smem, st, std::forward<Args>(args)...);
}

}  // namespace bs
