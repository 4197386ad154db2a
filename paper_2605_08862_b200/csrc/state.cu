// state.cu — rollout slot state: begin (Alg. 1 line 1), commit (lines 15/22 "y <- y o a"),
// state read-back, and pool staging append (per RL step).
#include "common.cuh"
#include "ctx.h"

namespace bs {

__global__ void begin_kernel(int n, int M, const int32_t* slots, const unsigned long long* uids,
                             const int32_t* prompt_ids, const int32_t* ptail, const int32_t* max_len,
                             int32_t* tail, int32_t* ctx_len, int32_t* pos, int32_t* ml,
                             int32_t* prompt, int32_t* finished, unsigned long long* uid) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    const int s = slots[b];
    int valid = 0;
    for (int i = M - 1; i >= 0; --i) {  // right-aligned; count the valid suffix
        const int t = ptail[(int64_t)b * M + i];
        tail[(int64_t)s * M + i] = t;
        if (t >= 0 && valid == M - 1 - i) ++valid;
    }
    ctx_len[s] = valid;
    pos[s] = 0;
    ml[s] = max_len[b];
    prompt[s] = prompt_ids[b];
    finished[s] = 0;
    uid[s] = uids[b];
    __threadfence();  // visible before a later launch's early plan reads it
}

// One warp per rollout (Alg. 1 lines 15/22): lane i owns tail slot i (M <= 32) and emitted
// token i (out_len <= k+1 <= 32); the shift of the tail is two shuffles.
__global__ void commit_kernel(int n, int M, int k, int eos, const int32_t* slots,
                              const int32_t* out_tokens, const int32_t* out_len, int32_t* tail,
                              int32_t* ctx_len, int32_t* pos, const int32_t* max_len,
                              int32_t* finished, int32_t* fin_out, int32_t* resp,
                              int64_t resp_stride) {
    pdl_wait();  // dependents launch at exit: a verify launch plans from this state early
    const int lane = threadIdx.x & 31;
    const int b = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (b >= n) return;
    const int s = slots[b];
    const int no = out_len[b];
    const int fin = finished[s];
    const int p = pos[s], L = max_len[s];
    const int32_t* out = out_tokens + (int64_t)b * (k + 1);
    int32_t* tl = tail + (int64_t)s * M;
    int f = fin;
    if (no > 0 && !fin) {
        const int32_t old = (lane < M) ? tl[lane] : -1;
        const int32_t ot = (lane < no) ? out[lane] : -1;
        // new tail[i] = (old ++ out)[i + no]
        const int src = lane + no;
        const int32_t from_old = __shfl_sync(0xFFFFFFFFu, old, src & 31);
        const int32_t from_out = __shfl_sync(0xFFFFFFFFu, ot, (src - M) & 31);
        if (lane < M) tl[lane] = (src < M) ? from_old : from_out;
        if (resp && lane < no && p + lane < resp_stride) resp[(int64_t)s * resp_stride + p + lane] = ot;
        const int32_t last = __shfl_sync(0xFFFFFFFFu, ot, no - 1);
        f = ((eos >= 0 && last == eos) || p + no >= L) ? 1 : 0;
        if (lane == 0) {
            ctx_len[s] = min(M, ctx_len[s] + no);
            pos[s] = p + no;
            if (f) finished[s] = 1;
        }
    } else if (!fin) {  // out of length, or an empty block of a live rollout: an error stop
        // (a needed row or the draft was invalid, reading R0; the error word says which)
        f = 1;
        if (lane == 0) finished[s] = 1;
    }
    if (fin_out && lane == 0) fin_out[b] = f;
    __threadfence();  // visible before a later launch's early plan reads it
}

__global__ void state_kernel(int n, const int32_t* slots, const int32_t* pos,
                             const int32_t* finished, int32_t* pos_out, int32_t* fin_out) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n) return;
    const int s = slots[b];
    if (pos_out) pos_out[b] = pos[s];
    if (fin_out) fin_out[b] = finished[s];
}

// Number of unfinished rollouts among slots[0..n) (one CTA; the host's per-chunk done check).
__global__ void live_count_kernel(int n, const int32_t* slots, const int32_t* finished, int32_t* out) {
    __shared__ int wsum[32];
    int c = 0;
    for (int b = threadIdx.x; b < n; b += blockDim.x) c += finished[slots[b]] == 0;
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        int t = (threadIdx.x < (int)(blockDim.x >> 5)) ? wsum[threadIdx.x] : 0;
        t = __reduce_add_sync(0xFFFFFFFFu, t);
        if (threadIdx.x == 0) *out = t;
    }
}

__global__ void pool_append_kernel(int n_seqs, int64_t n_tokens, const int32_t* prompt_ids,
                                   const int64_t* seq_off, const int32_t* tokens, int64_t base_tok,
                                   int base_seq, int32_t* dst_tokens, int64_t* dst_off,
                                   int32_t* dst_prompt) {
    const int64_t off0 = seq_off[0];
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = gid; t < n_tokens; t += stride) dst_tokens[base_tok + t] = tokens[off0 + t];
    for (int64_t s = gid; s <= n_seqs; s += stride) {
        dst_off[base_seq + s] = base_tok + (seq_off[s] - off0);
        if (s < n_seqs) dst_prompt[base_seq + s] = prompt_ids[s];
    }
}

cudaError_t launch_begin(bs_ctx* ctx, int32_t n, const int32_t* slots,
                         const unsigned long long* uids, const int32_t* prompt_ids,
                         const int32_t* tail, const int32_t* max_len, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    begin_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, ctx->M, slots, uids, prompt_ids, tail, max_len,
                                                  ctx->tail.p, ctx->ctx_len.p, ctx->pos.p,
                                                  ctx->max_len.p, ctx->prompt.p, ctx->finished.p,
                                                  ctx->uid.p);
    return cudaGetLastError();
}

cudaError_t launch_commit(bs_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* out_tokens,
                          const int32_t* out_len, int32_t k, int32_t* finished, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    return launch_pdl(commit_kernel, dim3((n + 3) / 4), dim3(128), 0, st, n, ctx->M, k,
                      ctx->cfg.eos_id, slots, out_tokens, out_len, ctx->tail.p, ctx->ctx_len.p,
                      ctx->pos.p, (const int32_t*)ctx->max_len.p, ctx->finished.p, finished,
                      ctx->responses, ctx->resp_stride);
}

cudaError_t launch_state(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t* pos,
                         int32_t* finished, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    state_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, slots, ctx->pos.p, ctx->finished.p, pos, finished);
    return cudaGetLastError();
}

cudaError_t launch_live_count(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t* out, cudaStream_t st) {
    live_count_kernel<<<1, 256, 0, st>>>(n, slots, ctx->finished.p, out);
    return cudaGetLastError();
}

cudaError_t launch_pool_append(bs_ctx* ctx, int32_t n_seqs, const int32_t* prompt_ids,
                               const int64_t* seq_offsets, const int32_t* tokens,
                               int64_t n_tokens, cudaStream_t st) {
    Pool& P = ctx->staging;
    const int64_t work = std::max<int64_t>(n_tokens, (int64_t)n_seqs + 1);
    const int blocks = (int)std::min<int64_t>(4096, (work + 255) / 256);
    pool_append_kernel<<<std::max(blocks, 1), 256, 0, st>>>(n_seqs, n_tokens, prompt_ids, seq_offsets,
                                                            tokens, P.n_tokens, P.n_seqs, P.tokens.p,
                                                            P.seq_off.p, P.seq_prompt.p);
    return cudaGetLastError();
}

}  // namespace bs
