// ngram.cu — draft-source variant: the n-gram linear-scan drafter (the paper's
// ablation baseline, "an n-gram-style scheme that performs pattern matching directly over
// raw token sequences", Table 7 at P:389-401).
//
// Reading N1: the anchor is the longest suffix y[-n:], n in [n_min, min(n_max,
// |y|, M)], occurring in the rollout's prompt pool followed by >= 1 token; among its occurrences
// the first in pool order (sequence index, then position) wins; the draft is the <= k tokens
// after it in its own sequence (clamped to max_len - pos - 1 like the suffix lookup, L6).  No
// counts and no index: the work is linear in the prompt's pool, which is the cost the paper
// attributes to n-gram matching.
//
// One CTA per rollout.  Thread t tests pool positions e = start + t, start + t + 256, ... of
// each of the prompt's sequences: the backward match length of T[..e] against the context
// (almost always 0 or 1 compare), keyed (n << 40 | (2^40 - 1 - e)) so that one max-reduction
// picks the longest match and, among equals, the earliest position.  Sequences are scanned in
// index order, and their token ranges are increasing in the sealed pool, so the earliest
// position is the earliest in pool order.  The sealed pool is read through the device-resident
// index descriptor, so captured graphs stay valid across seals (as lookup_kernel).
#include "lookup.cuh"

namespace bs {

constexpr int NG_NT = 256;

__global__ void __launch_bounds__(NG_NT) ngram_kernel(const LookupArgs a, int n_min, int n_max) {
    pdl_wait();
    __shared__ int32_t y[32];  // y[i] = y[-1-i] (the rollout's last M tokens)
    __shared__ unsigned long long wbest[NG_NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = blockIdx.x;
    const int slot = a.slots[b];
    const IndexDesc x = *a.desc;
    const bool stale = x.step != *a.cur_step;
    const int M = a.M;
    const int L = a.ctx_len[slot];
    const int P = a.prompt[slot];
    const int p = a.pos[slot], ml = a.max_len[slot];
    const bool fin = a.finished[slot] != 0 || p >= ml || stale;
    if (tid < M) y[tid] = a.tail[(int64_t)slot * M + (M - 1 - tid)];
    __syncthreads();
    const int nmax = min(min(n_max, M), L);
    constexpr unsigned long long PMASK = (1ull << 40) - 1ull;
    unsigned long long best = 0;
    if (!fin && nmax >= n_min) {
        const int y0 = y[0];
        for (int s = 0; s < x.n_seqs; ++s) {
            if (x.seq_prompt[s] != P) continue;  // uniform across the CTA
            const int64_t s0 = x.seq_off[s], s1 = x.seq_off[s + 1];
            for (int64_t e = s0 + tid; e + 1 < s1; e += NG_NT) {  // e + 1 < s1: a token follows
                if (__ldg(x.T + e) != y0) continue;
                int n = 1;
                while (n < nmax && e - n >= s0 && __ldg(x.T + e - n) == y[n]) ++n;
                if (n >= n_min) best = max(best, ((unsigned long long)n << 40) | (PMASK - (unsigned long long)e));
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
    if (lane == 0) wbest[warp] = best;
    __syncthreads();
    if (warp == 0) {
        best = (lane < NG_NT / 32) ? wbest[lane] : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
        int n = (int)(best >> 40), q = 0;
        int64_t e = 0, end = 0;
        if (best) {
            e = (int64_t)(PMASK - (best & PMASK));
            // the occurrence's sequence end: the first offset above e (sequences are increasing)
            int lo = 0, hi = x.n_seqs;  // seq_off[lo] <= e < seq_off[hi]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (x.seq_off[mid] <= e) lo = mid;
                else hi = mid;
            }
            end = x.seq_off[lo + 1];
            q = (int)min((int64_t)a.k, end - e - 1);
            q = min(q, max(0, ml - p - 1));
        } else {
            n = 0;
        }
        if (lane < a.k) a.draft[(int64_t)b * a.k + lane] = (lane < q) ? __ldg(x.T + e + 1 + lane) : -1;
        if (lane == 0) {
            a.draft_len[b] = q;
            if (a.match_len) a.match_len[b] = n;
            if (stale) atomicOr(a.dev_err, DEV_STALE);
        }
    }
    __threadfence();
    pdl_trigger();
}

cudaError_t launch_lookup_ngram(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t k, int32_t n_min,
                                int32_t n_max, int32_t* draft, int32_t* draft_len, int32_t* match_len,
                                cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const LookupArgs a = lookup_args(ctx, n, slots, k, draft, draft_len, match_len);
    cudaError_t e = launch_pdl(ngram_kernel, dim3(n), dim3(NG_NT), 0, st, a, (int)n_min, (int)n_max);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace bs
