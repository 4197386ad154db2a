// ctx.h — internal context of libbubblespec (host side).  Not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/bubblespec.h"
#include "common.cuh"

namespace bs {

// Device statistics counters (bs_stats_read): decoding-step accounting of SPEC S:478-484.
enum : int {
    STAT_STEPS_SPEC = 0,     // verification steps (q >= 1)
    STAT_STEPS_PLAIN = 1,    // plain decoding steps (empty draft, Alg. 1 lines 4-7)
    STAT_EMIT_SPEC = 2,      // tokens emitted by verification steps
    STAT_EMIT_PLAIN = 3,     // tokens emitted by plain steps
    STAT_ACCEPTED = 4,       // accepted draft tokens
    STAT_PROPOSED = 5,       // proposed draft tokens
    STAT_ROWS_VERIFIED = 6,  // logits rows streamed by the verify kernel
    STAT_ROWS_NEEDED = 7,    // rows Alg. 1 needs (up to the first rejection / EOS)
    STAT_HIST = 8,           // emitted-per-verification-step histogram, bins 0..32
    STAT_HIST_BINS = 33,
    STAT_COUNT = STAT_HIST + STAT_HIST_BINS
};

// Control words of the verify kernel: next rollout to claim, number of live rollouts.
enum : int { VCTL_NEXT = 0, VCTL_NACTIVE = 1, VCTL_MODE = 2, VCTL_ROWS = 3 };
// Scheduler words of the cluster verify kernel (verify_cluster.cuh): static cursor,
// rollouts done, CTAs exited, launch epoch.  All but the epoch are zero between launches
// (the last CTA out resets them).
// SC_NLIVE / SC_PLANNED form one 64-bit word (live count low, planned count high).
enum : int {
    SC_STATIC = 8, SC_NLIVE = 10, SC_PLANNED = 11, SC_DONE = 13, SC_EXIT = 14, SC_EPOCH = 15,
    VCTL_WORDS = 16
};

// Per-rollout plan of one verify launch (cluster kernel), written by the planning warps at
// kernel start and published by its epoch tag (written last).
struct RollRec {
    int32_t q, slot, pos, tag;   // clamped draft length (-1: no rows), slot, position, epoch
    unsigned long long uid;
    long long rowno0;            // logits row of row 0
    int32_t d0, aligned0;        // d_1 (or -1), row 0 16-byte aligned
    int32_t pad[2];
};
static_assert(sizeof(RollRec) == 48, "RollRec layout");

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t want) {
        if (want <= n && p) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        size_t alloc = want ? want : 1;
        cudaError_t e = cudaMalloc(&p, alloc * sizeof(T));
        if (e == cudaSuccess) n = alloc;
        return e;
    }
    // Stream-ordered growth (cudaMallocAsync / cudaFreeAsync from the device's memory pool, which
    // bs_create keeps cached): no device-synchronising cudaMalloc / cudaFree on a per-RL-step path
    // (a synchronous re-allocation of the index table once stalled a seal for over a second).
    // Buffers grown this way must be released with release_async.
    cudaError_t ensure_async(size_t want, cudaStream_t st) {
        if (want <= n && p) return cudaSuccess;
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        n = 0;
        const size_t alloc = want ? want + want / 4 : 1;  // 25 % headroom: fewer regrowths
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), alloc * sizeof(T), st);
        if (e == cudaSuccess) n = alloc;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
};

// Stream-ordered scratch: cudaMallocAsync / cudaFreeAsync from the device's default memory
// pool (bs_create keeps freed pool memory cached), so per-RL-step builds never hit the
// synchronising cudaMalloc / cudaFree.  Freed (stream-ordered) when it goes out of scope.
template <typename T>
struct AsyncBuf {
    T* p = nullptr;
    cudaStream_t st = nullptr;
    cudaError_t alloc(size_t n, cudaStream_t s) {
        st = s;
        return cudaMallocAsync(reinterpret_cast<void**>(&p), (n ? n : 1) * sizeof(T), s);
    }
    AsyncBuf() = default;
    AsyncBuf(const AsyncBuf&) = delete;
    AsyncBuf& operator=(const AsyncBuf&) = delete;
    ~AsyncBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

struct IndexEntry;
// The sealed index as the lookup kernel sees it (device-resident; bs_draft_pool_seal updates it).
struct IndexDesc {
    IndexEntry* table;
    uint64_t mask;
    const int32_t* T;
    const int32_t* seq_start_of;
    unsigned long long step;  // the rl_step this index was sealed for (~0: none / failed seal)
    // the sealed pool as the n-gram drafter scans it (bs_draft_lookup_ngram)
    const int64_t* seq_off;     // [n_seqs + 1] offsets into T
    const int32_t* seq_prompt;  // [n_seqs]
    int32_t n_seqs;
};

struct Pool {
    DevBuf<int32_t> tokens;
    DevBuf<int64_t> seq_off;  // absolute offsets into tokens, n_seqs + 1
    DevBuf<int32_t> seq_prompt;
    int64_t n_tokens = 0;
    int32_t n_seqs = 0;
    uint64_t step = 0;
    bool valid = false;
};

}  // namespace bs

struct bs_ctx {
    bs_config cfg;
    int S = 0;  // mass shift (reading R4)
    int M = 0;  // match_max
    uint64_t tau_q = 0;  // confidence threshold round(min_token_prob * 2^32) for the next seal (C1)
    std::string err;
    int num_sms = 148;
    int verify_kind = 0;  // bsx_set_verify_kernel (0: auto)
    int early_plan = 0;   // bsx_set_early_plan: the verify launch may plan before its PDL wait
    int max_clusters = 0; // bsx_set_max_clusters: cap on the cluster verify grid (0: all resident)
    const unsigned long long* rs_key = nullptr;  // bsx_set_row_stats (LM-head epilogue row statistics)
    const uint32_t* rs_bad = nullptr;
    // per-context (hence per-device) kernel launch setup, done once on this ctx's device:
    // dynamic shared memory attributes set, and the cluster kernel's resident cluster count
    size_t kcfg_cluster_smem = 0, kcfg_split_smem = 0;
    int kcfg_clusters = 0, kcfg_topp = 0, kcfg_rows = 0;
    int kcfg_coop = -1;  // cooperative cluster launches: -1 untested, 0 unsupported, 1 used
    int env_kind = 0, env_eager = 1;  // BS_VERIFY_KERNEL / BS_NO_EAGER, BS_FORCE_EAGER (tools), read at create
    // rollout slots
    bs::DevBuf<int32_t> tail;  // [R, M] right-aligned context tail
    bs::DevBuf<int32_t> ctx_len, pos, max_len, prompt, finished;
    bs::DevBuf<unsigned long long> uid;
    bs::DevBuf<uint32_t> dev_err;
    // pools: staging (being assembled) and sealed (indexed)
    bs::Pool staging, sealed;
    bs::DevBuf<int32_t> seq_start_of, seq_end_of, prompt_of;  // per sealed pool token
    bs::DevBuf<bs::IndexEntry> table;
    uint64_t table_mask = 0;
    bs::DevBuf<bs::IndexDesc> idx_desc;
    // the rl_step of the latest put / exchange / seal (device word): a lookup whose index was
    // sealed for another step is stale, checked on the device so that replayed
    // CUDA graphs are covered too
    bs::DevBuf<unsigned long long> cur_step;
    // verify scratch: clamped q per rollout, the step's row table (RowDesc, 48 B per row)
    // and its control words
    bs::DevBuf<int32_t> rb_q, vqueue;
    bs::DevBuf<unsigned int> vctl;
    // per verified row (b*(k_max+1)+j): status, candidate token, Z, fp32 normaliser
    bs::DevBuf<int32_t> vrow_status, vrow_cand;
    bs::DevBuf<unsigned long long> vrow_z;
    bs::DevBuf<float> vrow_norm;
    // per rollout: lowest deciding row seen (claim hint) and the state word (rows done |
    // rows deciding << 32)
    bs::DevBuf<int32_t> vroll_first;
    bs::DevBuf<unsigned long long> vroll_state;
    // cluster-kernel scheduler: per-rollout claim counter (epoch << 32 | next unclaimed
    // row) and per-rollout plan records
    bs::DevBuf<unsigned long long> vnext_row;
    bs::DevBuf<bs::RollRec> vrrec;
    bs::DevBuf<unsigned long long> vlive;  // live rollouts (epoch << 32 | b), compacted by the planners
    bs::DevBuf<unsigned long long> stats;  // STAT_COUNT counters
    int32_t* responses = nullptr;           // optional [max_rollouts, resp_stride] output
    int64_t resp_stride = 0;
};

namespace bs {
// launchers implemented in the .cu files
struct LookupArgs;
LookupArgs lookup_args(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t k, int32_t* draft,
                       int32_t* draft_len, int32_t* match_len);
// committed / looked_up (optional): set when the launch also committed (bs_verify_commit) /
// also looked up the next step's drafts described by `lookup` (bs_verify_commit_lookup)
cudaError_t launch_verify(bs_ctx* ctx, int32_t n, const int32_t* slots, const void* logits,
                          const int64_t* row_index, int64_t stride, const int32_t* draft,
                          const int32_t* draft_len, int32_t k, float T, float top_p, int32_t top_k,
                          int32_t* out_tokens, int32_t* out_len, int32_t* out_acc,
                          float* out_norm, unsigned long long* out_z, cudaStream_t st,
                          int32_t* commit_finished = nullptr, bool* committed = nullptr,
                          const LookupArgs* lookup = nullptr, bool* looked_up = nullptr);
cudaError_t launch_lookup(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t k,
                          int32_t* draft, int32_t* draft_len, int32_t* match_len,
                          cudaStream_t st);
cudaError_t launch_lookup_ngram(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t k, int32_t n_min,
                                int32_t n_max, int32_t* draft, int32_t* draft_len, int32_t* match_len,
                                cudaStream_t st);
cudaError_t seal_index(bs_ctx* ctx, cudaStream_t st, std::string& why);
// device word cur_step <- step (the latest put / exchange / seal; staleness)
cudaError_t set_cur_step(bs_ctx* ctx, uint64_t step, cudaStream_t st);
// publish the index descriptor with no sealed step (every lookup is stale until a seal)
void invalidate_index(bs_ctx* ctx, cudaStream_t st);
cudaError_t launch_commit(bs_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* out_tokens,
                          const int32_t* out_len, int32_t k, int32_t* finished, cudaStream_t st);
cudaError_t launch_begin(bs_ctx* ctx, int32_t n, const int32_t* slots,
                         const unsigned long long* uids, const int32_t* prompt_ids,
                         const int32_t* tail, const int32_t* max_len, cudaStream_t st);
cudaError_t launch_live_count(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t* out, cudaStream_t st);
cudaError_t launch_state(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t* pos,
                         int32_t* finished, cudaStream_t st);
cudaError_t launch_pool_append(bs_ctx* ctx, int32_t n_seqs, const int32_t* prompt_ids,
                               const int64_t* seq_offsets, const int32_t* tokens,
                               int64_t n_tokens, cudaStream_t st);
cudaError_t launch_synth_bank(void* bank, int64_t rows, int32_t V, uint32_t seed, float beta,
                              cudaStream_t st);
cudaError_t launch_target_rows(bs_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* draft,
                               const int32_t* draft_len, int32_t k, uint32_t tseed, int32_t mode,
                               int64_t nbank, int64_t* row_index, cudaStream_t st);
}  // namespace bs
