/*
 * bubblespec.h — C-ABI of the B200-native BubbleSpec hot path (arXiv 2605.08862).
 *
 * The calls follow the paper's problem statement, Alg. 1:
 * inputs are the prompt, the target policy's logits, the suffix index built from
 * the pre-generated token pools and the maximum length L.  One decoding
 * step of a batch of rollouts is
 *
 *     bs_draft_lookup  ->  [engine forward produces logits rows]  ->  bs_verify_step  ->  bs_commit
 *
 * and once per RL step the pools pre-generated in the inter-GPU bubbles
 * are put, optionally exchanged across DP ranks by prompt id (P:199,
 * P:346), and sealed (index build).
 *
 * Conventions (all functions):
 *  - Every array argument is a DEVICE pointer owned by the caller, unless stated.
 *    The library owns pools, the index, per-slot rollout state and scratch.
 *  - Every call is stream-ordered and asynchronous on `stream` (a cudaStream_t
 *    passed as void*; NULL = legacy default stream).  One bs_ctx must be driven
 *    from one stream at a time; a bs_ctx is not thread-safe (one per GPU / rank).
 *  - Device: a call on a bs_ctx (or a bs_bubble_sync) runs on that object's device
 *    and restores the caller's current device before it returns; the context-free
 *    calls (bs_unified_attention, bs_lm_head_logits) run on the caller's current
 *    device, which must hold their pointers and `stream`.
 *  - Host-side argument validation returns a bs_status synchronously and never
 *    throws; bs_last_error() gives the text.  Device-side anomalies (NaN / +inf
 *    logits, an all -inf row, |max logit / T| too large, draft id outside [0, V),
 *    index key collision) set a sticky device error word that bs_sync_status()
 *    reports and clears.
 *  - Randomness: the only random numbers are Philox4x32-10 draws with
 *    key = config.seed and counter = (position, purpose, uid_lo, uid_hi), where
 *    position = generated-token index, purpose 0 = ACCEPT, 1 = SAMPLE, and uid
 *    is the rollout's global id (reading R6).  Results are therefore
 *    independent of batching, slot assignment and DP sharding.
 *  - Arithmetic: decisions are made in the reference arithmetic R of DESIGN.md §3
 *    (integer masses, exact sums), so outputs are bit-identical to the CPU oracle.
 */
#ifndef BUBBLESPEC_H_
#define BUBBLESPEC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bs_ctx bs_ctx;

typedef enum {
    BS_OK = 0,
    BS_ERR_INVALID = 1,   /* bad argument (host-side check)                       */
    BS_ERR_OOM = 2,       /* device allocation failed                             */
    BS_ERR_CUDA = 3,      /* a CUDA runtime call failed (no GPU, launch error ...) */
    BS_ERR_STALE = 4,     /* lookup against a pool sealed for another rl_step     */
    BS_ERR_CAPACITY = 5,  /* pool / slot capacity exceeded                        */
    BS_ERR_NCCL = 6,      /* NCCL unavailable or a collective failed              */
    BS_ERR_DEVICE = 7     /* device error word set (see bs_sync_status)           */
} bs_status;

/* Device error word bits (bs_sync_status). */
#define BS_DEV_BAD_LOGIT   0x1u  /* NaN or +inf logit in a verified row (reading R0)   */
#define BS_DEV_ALL_NEGINF  0x2u  /* a verified row is all -inf (reading R0)            */
#define BS_DEV_RANGE       0x4u  /* |fl(m * log2e/T)| >= 2^24 (reading R0)              */
#define BS_DEV_BAD_DRAFT   0x8u  /* draft token outside [0, V)                          */
#define BS_DEV_INDEX_KEY   0x10u /* 64-bit key collision between two index windows      */
#define BS_DEV_STALE       0x20u /* a lookup ran while the index was stale: pools were put  */
                                 /* for a newer rl_step than the one sealed;  */
                                 /* its drafts are empty; bs_sync_status -> BS_ERR_STALE   */

typedef struct {
    int32_t vocab;                /* V in [1, 524288]: logits row length                */
    int32_t eos_id;               /* EOS token id, or -1 for none (Alg. 1) */
    int32_t k_max;                /* max draft block length K, 1..31 (P:299 uses 4)    */
    int32_t match_max;            /* M, max anchor length, 1..32 (reading L1)          */
    int32_t match_min;            /* L_min >= 1, min anchor length              */
    int32_t max_rollouts;         /* number of rollout slots, in [1, 2097151]           */
    int64_t pool_capacity_tokens; /* pool token capacity per RL step                    */
    int32_t pool_capacity_seqs;   /* pool sequence capacity per RL step                 */
    int32_t device;               /* CUDA device ordinal                                */
    uint64_t seed;                /* Philox key (reading R6)                            */
} bs_config;

typedef struct {
    float temperature; /* T >= 0; T == 0 is greedy (argmax, lowest id)          */
    float top_p;       /* (0, 1]; nucleus over integer masses (reading R5)     */
    int32_t top_k;     /* >= 0; 0 = off.  Keep the top_k heaviest masses, tie-closed  */
                       /* (reading R5k, "any top-p/top-k filtering"), applied   */
                       /* before top-p.  Ignored when T == 0 (greedy).     */
} bs_sampling;

/* ---------------------------------------------------------------- lifetime */
/* Allocate a context on config->device.  Returns BS_ERR_INVALID for an invalid
 * config, BS_ERR_CUDA if no device, BS_ERR_OOM on allocation failure. */
bs_status bs_create(const bs_config* config, bs_ctx** out);
void bs_destroy(bs_ctx* ctx);
/* Text of the last host-side error of this ctx (or of the last bs_create if ctx is NULL). */
const char* bs_last_error(const bs_ctx* ctx);
/* Synchronise `stream`, read and clear the device error word.  Writes the word to
 * *word (may be NULL); returns BS_ERR_DEVICE if it was non-zero. */
bs_status bs_sync_status(bs_ctx* ctx, void* stream, uint32_t* word);
/* Library version string. */
const char* bs_version(void);

/* ---------------------------------------------------------------- rollouts */
/* Start n rollouts (Alg. 1 line 1: y <- x_{1:m}).
 *   slots[n]        slot index in [0, max_rollouts)
 *   uids[n]         globally unique rollout id (Philox counter words 2-3)
 *   prompt_ids[n]   prompt id; selects the pool used by lookup
 *   prompt_tail[n*M] the last M prompt tokens, right-aligned, -1 = padding on the left;
 *                   at least one valid token per rollout
 *   max_len[n]      L: maximum number of generated tokens (Alg. 1 "while |y| < L")
 * Resets pos = 0, finished = 0. */
bs_status bs_rollout_begin(bs_ctx* ctx, int32_t n, const int32_t* slots, const uint64_t* uids,
                           const int32_t* prompt_ids, const int32_t* prompt_tail,
                           const int32_t* max_len, void* stream);

/* Read per-slot state (device outputs, any may be NULL): pos[n], finished[n]. */
bs_status bs_rollout_state(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t* pos,
                           int32_t* finished, void* stream);

/* live[0] (device int32) = how many of slots[0..n) are not finished (one kernel; stream-ordered,
 * graph-capturable): the caller's "all rollouts done?" check without a host-side reduction. */
bs_status bs_rollout_live(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t* live, void* stream);

/* Bind (or unbind with NULL) a caller-owned device buffer [max_rollouts, stride]:
 * bs_commit then also writes every emitted token of slot s at responses[s*stride + t]
 * (t = generated-token index, t < stride), i.e. the rollout y of Alg. 1. */
bs_status bs_rollout_bind_output(bs_ctx* ctx, int32_t* responses, int64_t stride);

/* Copy the first n (<= 41) device statistics counters to HOST memory out[n] and
 * optionally reset them.  Counters (SPEC S:478-484 accounting): 0 verification steps
 * (q >= 1), 1 plain steps (q = 0), 2 tokens emitted by verification steps, 3 tokens
 * emitted by plain steps, 4 accepted drafts, 5 proposed drafts, 6 logits rows read by
 * the verify kernel, 7 rows Alg. 1 needs (up to the first rejection / EOS),
 * 8 + e (e = 0..32) verification steps that emitted e tokens.  Synchronises `stream`. */
bs_status bs_stats_read(bs_ctx* ctx, uint64_t* out, int32_t n, int32_t reset, void* stream);

/* ---------------------------------------------------------------- pools (per RL step) */
/* Append n_seqs pre-generated sequences to the pool being assembled for rl_step
 * ("prompt-associated token pools").  If rl_step differs from
 * the step being assembled, the staging pool is cleared first.
 *   prompt_ids[n_seqs]      owning prompt of each sequence
 *   seq_offsets[n_seqs+1]   offsets into tokens (offsets[0] may be non-zero)
 *   tokens[...]             token ids in [0, V)
 *   n_tokens                host copy of seq_offsets[n_seqs] - seq_offsets[0]
 * Returns BS_ERR_CAPACITY if the pool capacity would be exceeded. */
bs_status bs_draft_pool_put(bs_ctx* ctx, uint64_t rl_step, int32_t n_seqs,
                            const int32_t* prompt_ids, const int64_t* seq_offsets,
                            const int32_t* tokens, int64_t n_tokens, void* stream);

/* Build the draft index over the assembled pool for rl_step (the
 * suffix index of §3.2 bounded to depth M+K).  Synchronises
 * `stream` internally (per RL step, off the decode path).  Lookups against
 * another rl_step then return BS_ERR_STALE. */
bs_status bs_draft_pool_seal(bs_ctx* ctx, uint64_t rl_step, void* stream);

/* Confidence-scored drafts (draft-source variant; "candidate tokens with
 * higher confidence based on token node occurrence frequencies"; reading C1): from
 * the NEXT bs_draft_pool_seal on, the greedy descent of every draft stops before a token whose
 * empirical probability cnt(w c) / cnt(w) in the prompt's pool is below min_token_prob (cnt(w)
 * counts every occurrence of the current window w, also those ending a sequence), compared
 * exactly as cnt(w c) * 2^32 < round(min_token_prob * 2^32) * cnt(w).  The anchor is chosen as
 * before; a low-confidence first token gives an empty draft.  0 (the default) is the plain
 * greedy descent.  Host-only (no stream work).  BS_ERR_INVALID unless 0 <= min_token_prob <= 1. */
bs_status bs_draft_set_min_token_prob(bs_ctx* ctx, float min_token_prob);

/* Cross-rank draft exchange: all-gather the staging pools of all
 * ranks of `nccl_comm` (an ncclComm_t of world size R, this rank = rank) and keep
 * only sequences whose prompt_id % R == rank.  Replaces the staging pool with the
 * routed one; call bs_draft_pool_seal afterwards.  Returns BS_ERR_NCCL if NCCL
 * cannot be loaded.  Synchronises `stream`. */
bs_status bs_draft_exchange(bs_ctx* ctx, void* nccl_comm, int32_t rank, int32_t world,
                            uint64_t rl_step, void* stream);
/* Host-only routing plan used by bs_draft_exchange (no GPU needed).  Given the
 * all-gathered per-rank metadata — counts[2*world] = (n_seqs_r, n_tokens_r),
 * offs_all[world*(max_seqs+1)] (rank r's offsets, relative to its token segment, at
 * r*(max_seqs+1)) and prompts_all[world*max_seqs] — list, in (rank, seq) order, the
 * sequences this rank owns (prompt % world == rank): source position in the gathered
 * token buffer (r*max_tokens + offset), destination offset, length, prompt id.
 * Output arrays hold >= sum_r n_seqs_r entries (host memory).  Returns 0, or 1 on
 * inconsistent input. */
int bs_route_plan(int32_t world, int32_t rank, const int64_t* counts, const int64_t* offs_all,
                  const int32_t* prompts_all, int64_t max_seqs, int64_t max_tokens,
                  int64_t* plan_src, int64_t* plan_dst, int64_t* plan_len, int32_t* plan_prompt,
                  int32_t* nkeep, int64_t* ntok);
/* Helper: ncclGetUniqueId into a 128-byte host buffer (for bootstrapping a comm). */
bs_status bs_nccl_unique_id(void* id128);
/* Helper: ncclCommInitRank from a 128-byte unique id; *comm_out receives the ncclComm_t. */
bs_status bs_nccl_comm_init(void** comm_out, const void* id128, int32_t world, int32_t rank);
bs_status bs_nccl_comm_destroy(void* comm);

/* ---------------------------------------------------------------- bubble pre-generation */
/* Polling synchronizer of rollout pre-generation ("during the
 * pre-generation of B_{t+1}, each rank queries a central synchronizer every T decoding steps.
 * If the synchronizer reports that all ranks have completed B_t, pre-generation is halted";
 * T = 50).  It is an array of BS_BUBBLE_MAX_RANKS 64-bit words in the owner rank's
 * device memory (one per DP rank: the latest rl_step that rank finished, ~0 before any),
 * mapped into the other ranks' address spaces over NVLink by CUDA IPC.  Arrive and poll are
 * single-kernel, stream-ordered calls (capturable in a CUDA graph with the pre-generation
 * steps): no collective, so a rank still decoding its batch never waits on the pollers.
 * Pre-generation itself is plain decoding (bs_verify_* with draft_len = 0) of the next RL
 * step's prompts in spare rollout slots; its responses become the next step's pools
 * (bs_draft_pool_put, then bs_draft_exchange routes them to their owner ranks). */
#define BS_BUBBLE_MAX_RANKS 64
typedef struct bs_bubble_sync bs_bubble_sync;
/* Owner side: allocate the words on `device` (all ~0). */
bs_status bs_bubble_sync_create(int32_t device, bs_bubble_sync** out);
/* Owner side: the 64-byte CUDA IPC handle of the words (host memory handle64[64]), to be sent to
 * the other ranks (e.g. over the torch process group). */
bs_status bs_bubble_sync_export(const bs_bubble_sync* sync, void* handle64);
/* Peer side: map the owner's words on this rank's `device` (NVLink peer access).  A process
 * cannot open its own handle: the owner uses the object bs_bubble_sync_create returned. */
bs_status bs_bubble_sync_open(int32_t device, const void* handle64, bs_bubble_sync** out);
void bs_bubble_sync_destroy(bs_bubble_sync* sync);
/* Stream-ordered: after the work already on `stream` (the rank's last decoding step of B_t),
 * store rl_step into word `rank` (a system-scope release store).  rl_step != ~0. */
bs_status bs_bubble_sync_arrive(bs_bubble_sync* sync, int32_t rank, uint64_t rl_step, void* stream);
/* Stream-ordered: *halt (a device int32) = 1 if every word 0..world-1 holds >= rl_step (all
 * ranks completed B_t: stop pre-generating), else 0 (system-scope acquire loads). */
bs_status bs_bubble_sync_poll(bs_bubble_sync* sync, int32_t world, uint64_t rl_step, int32_t* halt,
                              void* stream);

/* ---------------------------------------------------------------- per decoding step */
/* Draft lookup (Alg. 1 line 3: "Retrieve a draft block from T using prefix y"):
 * anchor on the longest suffix (<= M) of each rollout's context that occurs in
 * its prompt's pool with a continuation, then descend greedily by occurrence
 * count (ties -> lowest id) for up to k tokens (readings L1-L6).
 *   slots[n]; outputs draft_tokens[n*k] (row b holds draft_len[b] tokens, rest -1),
 *   draft_len[n] (clamped to max_len - pos - 1, 0 if finished),
 *   match_len[n] (anchor length m*, 0 if none; may be NULL).
 * BS_ERR_STALE if the index is not sealed for rl_step; k in [0, k_max]. */
bs_status bs_draft_lookup(bs_ctx* ctx, uint64_t rl_step, int32_t n, const int32_t* slots,
                          int32_t k, int32_t* draft_tokens, int32_t* draft_len,
                          int32_t* match_len, void* stream);

/* Draft-source variant: the n-gram linear-scan drafter ("pattern
 * matching directly over raw token sequences", "a linear match of repeated token
 * sequences to return the candidate with the longest common prefix"; the paper's Table 7
 * ablation).  Reading N1: anchor on the longest suffix y[-n:] of the rollout's
 * context, n in [n_min, min(n_max, |y|)], that occurs in its prompt's sealed pool followed by a
 * token; the first such occurrence in pool order (sequence index, then position) gives the
 * draft: the up to k tokens after it in its sequence.  No index is used: the cost is linear in
 * the prompt's pool (one CTA per rollout).  Outputs as bs_draft_lookup (match_len = n, 0 if none;
 * draft_len clamped to max_len - pos - 1, 0 if finished).  Errors: BS_ERR_STALE as
 * bs_draft_lookup; BS_ERR_INVALID unless 1 <= n_min <= n_max <= match_max and 0 <= k <= k_max. */
bs_status bs_draft_lookup_ngram(bs_ctx* ctx, uint64_t rl_step, int32_t n, const int32_t* slots,
                                int32_t k, int32_t n_min, int32_t n_max, int32_t* draft_tokens,
                                int32_t* draft_len, int32_t* match_len, void* stream);

/* Lossless verification of one draft block per rollout (Eq. 2 P:203-205,
 * Eq. 3, Alg. 1, bonus P:308).  Pure: reads rollout state,
 * writes only its outputs.
 *   logits_bf16  bf16 logits rows of length V, row stride row_stride_elems (>= V)
 *   row_index    [n*(k+1)] int64 row numbers into logits_bf16, or NULL for the dense
 *                layout [n, k+1, V] (row b*(k+1)+j).  Row j of rollout b is the
 *                target distribution for generated-token index pos_b + j, i.e.
 *                after prefix y_b + d_1..d_j.  Rows j > draft_len[b] are not read.
 *   draft_tokens [n*k], draft_len[n] (values are clamped to [0, min(k, max_len-pos-1)])
 *   sampling     temperature / top-p of p_t
 * Outputs: out_tokens[n*(k+1)] emitted tokens (accepted drafts, then the recovered
 *   or bonus token unless an accepted EOS ended the block), out_len[n],
 *   out_accepted[n] accepted draft count, and (may be NULL) out_norm[n*(k+1)] the
 *   softmax normaliser sum_i exp((l_i - max)/T) of each verified row (fp32 from the
 *   exact integer sum) and out_z[n*(k+1)] the exact integer normaliser Z' of R.
 *   Entries of rows that were not needed are 0. */
bs_status bs_verify_step(bs_ctx* ctx, int32_t n, const int32_t* slots, const void* logits_bf16,
                         const int64_t* row_index, int64_t row_stride_elems,
                         const int32_t* draft_tokens, const int32_t* draft_len, int32_t k,
                         bs_sampling sampling, int32_t* out_tokens, int32_t* out_len,
                         int32_t* out_accepted, float* out_norm, uint64_t* out_z,
                         void* stream);

/* bs_verify_step followed by bs_commit, fused into one launch where the verify kernel
 * supports it (the cluster kernel, top_p = 1): the thread that finalizes a rollout's
 * step (Alg. 1 lines 10-31) also performs that rollout's commit (lines 15/22 "y <- y o a";
 * same state update as bs_commit), so no separate commit kernel runs.  Arguments are
 * those of bs_verify_step plus bs_commit's `finished` output [n] (may be NULL).  Results
 * and rollout state are identical to bs_verify_step + bs_commit (tested). */
bs_status bs_verify_commit(bs_ctx* ctx, int32_t n, const int32_t* slots, const void* logits_bf16,
                           const int64_t* row_index, int64_t row_stride_elems,
                           const int32_t* draft_tokens, const int32_t* draft_len, int32_t k,
                           bs_sampling sampling, int32_t* out_tokens, int32_t* out_len,
                           int32_t* out_accepted, float* out_norm, uint64_t* out_z,
                           int32_t* finished, void* stream);

/* bs_verify_commit followed by bs_draft_lookup for the NEXT decoding step (Alg. 1's loop:
 * the draft of step t+1 is the pool lookup from the context committed at step t),
 * fused into the same launch where bs_verify_commit is fused: the warp that commits a
 * rollout then looks up its next draft from the just-committed state (held in registers).
 *   draft_tokens / draft_len  IN: this step's drafts (as bs_verify_commit);
 *                             OUT: the next step's drafts for the same slots and k
 *                             (bs_draft_lookup's outputs), written in place
 *   match_len    [n] next-step anchored match length (may be NULL)
 *   rl_step      the index must be sealed for it (as bs_draft_lookup: BS_ERR_STALE)
 * Other arguments as bs_verify_commit.  Results, rollout state and next drafts are identical
 * to bs_verify_commit + bs_draft_lookup (tested); where the launch cannot fuse (top_p < 1, V
 * above the cluster kernel's limit) the separate kernels run. */
bs_status bs_verify_commit_lookup(bs_ctx* ctx, uint64_t rl_step, int32_t n, const int32_t* slots,
                                  const void* logits_bf16, const int64_t* row_index,
                                  int64_t row_stride_elems, int32_t* draft_tokens, int32_t* draft_len,
                                  int32_t k, bs_sampling sampling, int32_t* out_tokens, int32_t* out_len,
                                  int32_t* out_accepted, float* out_norm, uint64_t* out_z,
                                  int32_t* finished, int32_t* match_len, void* stream);

/* Commit (Alg. 1 lines 15/22 "y <- y o a"): append out_len[b] tokens of row b of
 * out_tokens [n*(k+1)] to each rollout, advance its position, and mark it
 * finished on an emitted EOS or when pos reaches max_len (Alg. 1 line 2).
 * finished[n] (may be NULL) receives the finished flags. */
bs_status bs_commit(bs_ctx* ctx, int32_t n, const int32_t* slots, const int32_t* out_tokens,
                    const int32_t* out_len, int32_t k, int32_t* finished, void* stream);

/* ---------------------------------------------------------------- unified attention (f2) */
/* Unified variable-query-length decode attention (Table 2 at
 * P:220-232): one launch over a batch mixing plain decode requests (q_len = 1) and speculative
 * requests (q_len = 1 + drafts), causal grouped-query attention over a paged bf16 KV cache,
 * the short-query matmuls on the tensor cores (tcgen05, TMEM accumulators, TMA-loaded KV).
 *   q            [T, H_q, head_dim] bf16, T = sum_b q_len[b]; request b's rows follow request
 *                b-1's (b = 0 first); its q_len[b] tokens are the LAST of its context
 *   k_cache/v_cache [num_pages, H_kv, page_size, head_dim] bf16 (device)
 *   page_table   [B, max_pages] int32 (device): page of tokens [i*page_size, (i+1)*page_size)
 *   ctx_len_dev  [B] int32 (device) and ctx_len / q_len [B] (HOST copies: the launch plan)
 *   scale        softmax scale (<= 0: 1/sqrt(head_dim))
 *   out          [T, H_q, head_dim] bf16: softmax(q k^T * scale, causal) v, token i of request b
 *                attending keys 0 .. ctx_len[b] - q_len[b] + i, query head h using KV head
 *                h / (H_q / H_kv)
 *   workspace    device scratch of bs_unified_attention_workspace() bytes; the call builds
 *                its work units (request, KV head, key-tile range) on the host from ctx_len /
 *                q_len and copies them into the workspace on `stream` from pageable memory, so
 *                it is not CUDA-graph capturable (capture the decode loop around it instead)
 * Supported: head_dim = 128, page_size = 64, q_len[b] * H_q / H_kv <= 128.  Errors:
 * BS_ERR_INVALID (shapes), BS_ERR_CAPACITY (workspace too small), BS_ERR_CUDA. */
bs_status bs_unified_attention_workspace(int32_t B, const int32_t* ctx_len, const int32_t* q_len, int32_t H_q,
                                         int32_t H_kv, int64_t* bytes);
bs_status bs_unified_attention(const void* q, const void* k_cache, const void* v_cache, int64_t num_pages,
                               const int32_t* page_table, int32_t max_pages, const int32_t* ctx_len_dev,
                               const int32_t* ctx_len, const int32_t* q_len, int32_t B, int32_t H_q, int32_t H_kv,
                               int32_t head_dim, int32_t page_size, float scale, void* out, void* workspace,
                               int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- LM head + fused row statistics (f3) */
/* The target policy's logits from the last hidden states, on the tensor cores, with the
 * verify's first pass fused into the GEMM epilogue:
 *   logits[r, v] = bf16(sum_k h[r, k] * W[v, k])  (fp32 accumulation, round to nearest even)
 *   row_key[r]   = (order key of max_v logits[r, v]) << 32 | (0xFFFFFFFF - lowest argmax)
 *                  (order key of bf16 bits b: b | 0x8000 if b >= 0 else ~b & 0xFFFF; NaN excluded)
 *   row_bad[r]   = 1 if a NaN or +inf logit occurred (reading R0)
 * h [rows, d] and W [V, d] bf16 row-major (16-byte aligned), d a multiple of 64; logits row stride
 * ld_logits >= V elements.  Errors: BS_ERR_INVALID, BS_ERR_CUDA. */
bs_status bs_lm_head_logits(const void* h, const void* w, int32_t rows, int32_t d, int32_t V, void* logits,
                            int64_t ld_logits, uint64_t* row_key, uint32_t* row_bad, void* stream);
/* Give the verify launches of this ctx the row statistics of bs_lm_head_logits (indexed like the
 * logits rows the verify reads); the cluster verify kernel then skips its max pass.  Results are
 * identical (tested).  NULL, NULL clears.  The arrays must describe the logits of every verify call
 * made while set. */
bs_status bsx_set_row_stats(bs_ctx* ctx, const uint64_t* row_key, const uint32_t* row_bad);

/* ---------------------------------------------------------------- tuning */
/* Select the kernel bs_verify_step uses for rows without top-p (all compute identical
 * results): 0 auto (= 3 when ceil(V/8) <= 53248, else 1; env BS_VERIFY_KERNEL
 * overrides auto), 1 one CTA per row (rows streamed twice through a TMA ring), 3 pipelined
 * 8-CTA cluster (row slices resident in shared memory, max and mass passes overlapped across
 * rows).  Takes effect for calls enqueued (or graphs captured) after it.  Errors:
 * BS_ERR_INVALID on a NULL ctx or an unknown kind (2, the former unpipelined split kernel, is
 * no longer accepted). */
bs_status bsx_set_verify_kernel(bs_ctx* ctx, int32_t kind);

/* Programmatic dependent launch (PDL) contract of the verify launches.  With on = 1 the
 * caller promises that the kernel enqueued immediately before a bs_verify_* call on its
 * stream writes none of the verify's plan inputs (slots, draft_tokens, draft_len) nor any
 * rollout state (it may write the logits and row_index: those are read only after the
 * launch's griddepcontrol.wait); the launch then plans its rollouts before that wait,
 * overlapping the preceding kernel (the model forward).  RolloutEngine's decode step (target
 * rows -> verify) keeps that contract.  Default 0: every read follows the wait.  Errors:
 * BS_ERR_INVALID on a NULL ctx or on not in {0, 1}. */
bs_status bsx_set_early_plan(bs_ctx* ctx, int32_t on);

/* Cap the cluster verify kernel's grid at max_clusters 8-CTA clusters (0 = every cluster that
 * can be resident, the default).  Lets several contexts (e.g. rollout groups on separate
 * streams) run their verify launches concurrently on one GPU.  Takes effect for calls enqueued
 * (or graphs captured) after it.  Errors: BS_ERR_INVALID on a NULL ctx or max_clusters < 0. */
bs_status bsx_set_max_clusters(bs_ctx* ctx, int32_t max_clusters);

/* Diagnostics (host memory out[n]): 0 resident clusters of the cluster verify kernel (0 until
 * its first launch), 1 cooperative launch in use (-1 untested, 0 no, 1 yes), 2 SM count,
 * 3 early plan.  Returns the number of values written. */
int32_t bsx_launch_info(const bs_ctx* ctx, int64_t* out, int32_t n);

/* ---------------------------------------------------------------- synthetic workload */
/* Not part of the method: device twins of workloads/synth.py so a
 * multi-GB logit bank need not be generated on the host.  Bit-identical to numpy. */
/* bank[rows, V] bf16: Irwin-Hall(4 hashed bytes) * 2^-6; the peak column holds beta. */
bs_status bsx_synth_bank(void* bank_bf16, int64_t rows, int32_t V, uint32_t bank_seed,
                         float beta, void* stream);
/* out[i] (bf16), i < n: (sum of the 4 bytes of h32(i * 0x9E3779B1 + base) - 510) * mult, the
 * values of workloads/attn.py (bit-identical). */
bs_status bsx_synth_attn_values(void* out_bf16, int64_t n, uint32_t base, float mult, void* stream);
/* Synthetic target "forward": row_index[b*(k+1)+j] = target_row(prompt, pos+j, prev_j)
 * for j <= draft_len[b] (prev_0 = last context token, prev_j = draft[j-1]).
 * mode: 0 position, 1 markov, 2 mixed, 3 sample (workloads.TargetSpec). */
bs_status bsx_target_rows(bs_ctx* ctx, int32_t n, const int32_t* slots,
                          const int32_t* draft_tokens, const int32_t* draft_len, int32_t k,
                          uint32_t target_seed, int32_t mode, int64_t nbank,
                          int64_t* row_index, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BUBBLESPEC_H_ */
