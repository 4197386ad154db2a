// synth.cu — device twins of workloads/synth.py (synthetic inputs, NOT the method).
// Bit-identical to the numpy generators; checked by tests/test_gpu_synth.py.
#include <cuda_bf16.h>

#include "common.cuh"
#include "ctx.h"

namespace bs {

__device__ __forceinline__ uint16_t synth_elem(uint32_t hr, uint32_t col, int peak, float beta) {
    const uint32_t h = h32(hr ^ col);
    const int s = (int)(h & 255u) + (int)((h >> 8) & 255u) + (int)((h >> 16) & 255u) + (int)(h >> 24) - 510;
    float v = (float)s * 0.015625f;
    if ((int)col == peak) v = beta;
    const __nv_bfloat16 bv = __float2bfloat16_rn(v);
    uint16_t u;
    memcpy(&u, &bv, 2);
    return u;
}

__global__ void synth_bank_kernel(uint16_t* bank, int64_t rows, int V, uint32_t seed, float beta) {
    const uint32_t s0 = h32(seed);
    const uint32_t sp = h32(seed ^ 0x5BD1E995u);
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
        const uint32_t hr = h32(s0 ^ (uint32_t)r);
        const int peak = (int)(h32(sp ^ (uint32_t)(r >> 4)) % (uint32_t)V);  // peak groups of 16 rows
        uint16_t* out = bank + r * (int64_t)V;
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < V; c += gridDim.x * blockDim.x)
            out[c] = synth_elem(hr, (uint32_t)c, peak, beta);
    }
}

__global__ void target_rows_kernel(int n, int k, int M, const int32_t* slots, const int32_t* draft,
                                   const int32_t* draft_len, const int32_t* tail, const int32_t* pos,
                                   const int32_t* prompt, const unsigned long long* uid, uint32_t tseed,
                                   int mode, int64_t nbank, int64_t* row_index) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    const int s = slots[b];
    const int q = min(max(draft_len[b], 0), k);
    const uint32_t base = h32(h32(tseed) ^ (uint32_t)prompt[s]);
    int prev = tail[(int64_t)s * M + (M - 1)];
    for (int j = 0; j <= q; ++j) {
        if (j > 0) prev = draft[(int64_t)b * k + j - 1];
        const uint32_t t = (uint32_t)(pos[s] + j);
        const uint32_t pv = (uint32_t)(prev + 0x10000000);
        uint32_t h;
        if (mode == 0 || mode == 3) h = h32(base ^ t);
        else if (mode == 1) h = h32(base ^ pv);
        else h = h32(h32(base ^ t) ^ pv);
        int64_t r = (int64_t)(h % (uint32_t)nbank);
        if (mode == 3)  // "sample": the rollout's own row of the peak group (uid mod 16)
            r = (int64_t)(h % (uint32_t)(nbank / 16)) * 16 + (int64_t)(uid[s] & 15ull);
        row_index[(int64_t)b * (k + 1) + j] = r;
    }
}

cudaError_t launch_synth_bank(void* bank, int64_t rows, int32_t V, uint32_t seed, float beta,
                              cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    dim3 grid((unsigned)std::min<int64_t>(64, (V + 255) / 256), (unsigned)std::min<int64_t>(rows, 65535));
    synth_bank_kernel<<<grid, 256, 0, st>>>(static_cast<uint16_t*>(bank), rows, V, seed, beta);
    return cudaGetLastError();
}

cudaError_t launch_target_rows(bs_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* draft,
                               const int32_t* draft_len, int32_t k, uint32_t tseed, int32_t mode,
                               int64_t nbank, int64_t* row_index, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    return launch_pdl(target_rows_kernel, dim3((n + 127) / 128), dim3(128), 0, st, n, k, ctx->M,
                      slots, draft, draft_len, (const int32_t*)ctx->tail.p,
                      (const int32_t*)ctx->pos.p, (const int32_t*)ctx->prompt.p,
                      (const unsigned long long*)ctx->uid.p, tseed, mode, nbank, row_index);
}

}  // namespace bs
