// api.cu — the C-ABI of include/bubblespec.h: argument validation, context lifetime,
// and dispatch to the kernels.  No torch types anywhere in this library.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "ctx.h"
#include "lookup.cuh"

using namespace bs;

static thread_local std::string g_create_err;

static bs_status fail(bs_ctx* ctx, bs_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    else g_create_err = buf;
    return s;
}

static bs_status cuda_fail(bs_ctx* ctx, cudaError_t e, const char* where) {
    cudaGetLastError();  // clear sticky-less errors
    return fail(ctx, e == cudaErrorMemoryAllocation ? BS_ERR_OOM : BS_ERR_CUDA, "%s: %s", where,
                cudaGetErrorString(e));
}

#define CK(ctx, x, where)                                  \
    do {                                                   \
        cudaError_t e_ = (x);                              \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, where); \
    } while (0)

static inline cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

bs_status bsx_set_verify_kernel(bs_ctx* c, int32_t kind) {
    if (!c || kind < 0 || kind > 3 || kind == 2) return BS_ERR_INVALID;
    c->verify_kind = kind;
    return BS_OK;
}

bs_status bsx_set_early_plan(bs_ctx* c, int32_t on) {
    if (!c || on < 0 || on > 1) return BS_ERR_INVALID;
    c->early_plan = on;
    return BS_OK;
}

bs_status bsx_set_max_clusters(bs_ctx* c, int32_t max_clusters) {
    if (!c || max_clusters < 0) return BS_ERR_INVALID;
    c->max_clusters = max_clusters;
    return BS_OK;
}

bs_status bsx_set_row_stats(bs_ctx* c, const uint64_t* row_key, const uint32_t* row_bad) {
    if (!c || (!row_key) != (!row_bad)) return BS_ERR_INVALID;
    c->rs_key = reinterpret_cast<const unsigned long long*>(row_key);
    c->rs_bad = row_bad;
    return BS_OK;
}

int32_t bsx_launch_info(const bs_ctx* c, int64_t* out, int32_t n) {
    if (!c || !out || n < 1) return 0;
    const int64_t v[4] = {c->kcfg_clusters, c->kcfg_coop, c->num_sms, c->early_plan};
    const int m = n < 4 ? n : 4;
    for (int i = 0; i < m; ++i) out[i] = v[i];
    return m;
}

const char* bs_version(void) { return "bubblespec-b200 0.1 (sm_100a)"; }

const char* bs_last_error(const bs_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

bs_status bs_create(const bs_config* cfg, bs_ctx** out) {
    if (!cfg || !out) return fail(nullptr, BS_ERR_INVALID, "null argument");
    *out = nullptr;
    if (cfg->vocab < 1) return fail(nullptr, BS_ERR_INVALID, "vocab must be >= 1");
    if (cfg->k_max < 1 || cfg->k_max > 31) return fail(nullptr, BS_ERR_INVALID, "k_max must be in [1, 31]");
    if (cfg->match_max < 1 || cfg->match_max > 32)
        return fail(nullptr, BS_ERR_INVALID, "match_max must be in [1, 32]");
    if (cfg->match_min < 1) return fail(nullptr, BS_ERR_INVALID, "match_min must be >= 1");
    // (the verify launch packs planned / live / hot rollout counts into 21-bit fields)
    if (cfg->max_rollouts < 1 || cfg->max_rollouts > 2097151)
        return fail(nullptr, BS_ERR_INVALID, "max_rollouts must be in [1, 2097151]");
    if (cfg->pool_capacity_tokens < 0 || cfg->pool_capacity_seqs < 0)
        return fail(nullptr, BS_ERR_INVALID, "negative pool capacity");
    if (cfg->eos_id >= cfg->vocab) return fail(nullptr, BS_ERR_INVALID, "eos_id >= vocab");
    // the largest vocabulary every verify kernel supports: the rows kernel's 32 super-chunks
    // of 16384 elements and the top-p kernel's 2048 coarse bins of 256 (V <= 524288)
    if (cfg->vocab > 524288) return fail(nullptr, BS_ERR_INVALID, "vocab > 524288 is not supported");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, BS_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
    }
    if (cfg->device < 0 || cfg->device >= ndev) return fail(nullptr, BS_ERR_INVALID, "bad device ordinal");
    bs::DeviceScope dev_scope_(cfg->device);
    if (dev_scope_.err != cudaSuccess) return cuda_fail(nullptr, dev_scope_.err, "cudaSetDevice");
    bs_ctx* c = new bs_ctx();
    c->cfg = *cfg;
    c->S = mass_shift(cfg->vocab);
    c->M = cfg->match_max;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, cfg->device);
    {  // tool / experiment overrides, read once per context (not per launch)
        const char* s = getenv("BS_VERIFY_KERNEL");
        c->env_kind = s ? atoi(s) : 0;
        c->env_eager = getenv("BS_NO_EAGER") ? 0 : (getenv("BS_FORCE_EAGER") ? 2 : 1);
    }
    {  // per-RL-step scratch is stream-ordered from the default pool: keep freed memory cached
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, cfg->device) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    const size_t R = (size_t)cfg->max_rollouts;
    const size_t rows = R * (size_t)(cfg->k_max + 1);
    bool okk = c->tail.ensure(R * c->M) == cudaSuccess && c->ctx_len.ensure(R) == cudaSuccess &&
               c->pos.ensure(R) == cudaSuccess && c->max_len.ensure(R) == cudaSuccess &&
               c->prompt.ensure(R) == cudaSuccess && c->finished.ensure(R) == cudaSuccess &&
               c->uid.ensure(R) == cudaSuccess && c->dev_err.ensure(1) == cudaSuccess &&
               c->rb_q.ensure(R) == cudaSuccess && c->vqueue.ensure(rows * 12 + 64) == cudaSuccess &&
               c->vctl.ensure(VCTL_WORDS) == cudaSuccess &&
               c->vrow_status.ensure(rows) == cudaSuccess && c->vrow_cand.ensure(rows) == cudaSuccess &&
               c->vrow_z.ensure(rows) == cudaSuccess && c->vrow_norm.ensure(rows) == cudaSuccess &&
               c->vroll_first.ensure(R) == cudaSuccess && c->vroll_state.ensure(R) == cudaSuccess &&
               c->vnext_row.ensure(R) == cudaSuccess && c->vrrec.ensure(R) == cudaSuccess &&
               c->vlive.ensure(R) == cudaSuccess &&
               c->staging.tokens.ensure((size_t)cfg->pool_capacity_tokens) == cudaSuccess &&
               c->staging.seq_off.ensure((size_t)cfg->pool_capacity_seqs + 1) == cudaSuccess &&
               c->staging.seq_prompt.ensure((size_t)cfg->pool_capacity_seqs) == cudaSuccess &&
               c->sealed.tokens.ensure((size_t)cfg->pool_capacity_tokens) == cudaSuccess &&
               c->sealed.seq_off.ensure((size_t)cfg->pool_capacity_seqs + 1) == cudaSuccess &&
               c->sealed.seq_prompt.ensure((size_t)cfg->pool_capacity_seqs) == cudaSuccess &&
               c->table.ensure(2) == cudaSuccess && c->stats.ensure(STAT_COUNT) == cudaSuccess &&
               c->idx_desc.ensure(1) == cudaSuccess && c->cur_step.ensure(1) == cudaSuccess;
    if (!okk) {
        bs_destroy(c);
        cudaGetLastError();
        return fail(nullptr, BS_ERR_OOM, "device allocation failed");
    }
    cudaMemset(c->tail.p, 0xFF, R * c->M * sizeof(int32_t));
    cudaMemset(c->ctx_len.p, 0, R * sizeof(int32_t));
    cudaMemset(c->pos.p, 0, R * sizeof(int32_t));
    cudaMemset(c->max_len.p, 0, R * sizeof(int32_t));
    cudaMemset(c->prompt.p, 0, R * sizeof(int32_t));
    cudaMemset(c->uid.p, 0, R * sizeof(unsigned long long));
    // unused slots are finished (no rows, no drafts)
    cudaMemset(c->finished.p, 0, R * sizeof(int32_t));
    cudaMemset(c->dev_err.p, 0, sizeof(uint32_t));
    cudaMemset(c->vctl.p, 0, VCTL_WORDS * sizeof(unsigned int));
    cudaMemset(c->vnext_row.p, 0, R * sizeof(unsigned long long));
    cudaMemset(c->vlive.p, 0, R * sizeof(unsigned long long));
    {  // scheduler epoch starts at 1: zeroed claim counters (epoch 0) read as unplanned
        const unsigned int one = 1u;
        cudaMemcpy(c->vctl.p + SC_EPOCH, &one, sizeof one, cudaMemcpyHostToDevice);
    }
    cudaMemset(c->stats.p, 0, STAT_COUNT * sizeof(unsigned long long));
    cudaMemset(c->table.p, 0, 2 * sizeof(IndexEntry));
    cudaMemset(c->staging.seq_off.p, 0, sizeof(int64_t));
    cudaMemset(c->sealed.seq_off.p, 0, sizeof(int64_t));
    c->table_mask = 1;
    {
        bs::IndexDesc d = {c->table.p, 1, c->sealed.tokens.p, c->seq_start_of.p, ~0ull};
        cudaMemcpy(c->idx_desc.p, &d, sizeof d, cudaMemcpyHostToDevice);
        const unsigned long long none = ~0ull;  // no pool put / sealed yet
        cudaMemcpy(c->cur_step.p, &none, sizeof none, cudaMemcpyHostToDevice);
    }
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        bs_destroy(c);
        return cuda_fail(nullptr, e, "bs_create");
    }
    *out = c;
    return BS_OK;
}

void bs_destroy(bs_ctx* c) {
    if (!c) return;
    bs::DeviceScope dev_scope_(c->cfg.device);
    c->tail.release(); c->ctx_len.release(); c->pos.release(); c->max_len.release();
    c->prompt.release(); c->finished.release(); c->uid.release(); c->dev_err.release();
    c->staging.tokens.release(); c->staging.seq_off.release(); c->staging.seq_prompt.release();
    c->sealed.tokens.release(); c->sealed.seq_off.release(); c->sealed.seq_prompt.release();
    c->seq_start_of.release(); c->seq_end_of.release(); c->prompt_of.release();
    c->table.release(); c->idx_desc.release(); c->cur_step.release(); c->rb_q.release(); c->vqueue.release(); c->vctl.release();
    c->vrow_status.release(); c->vrow_cand.release(); c->vrow_z.release(); c->vrow_norm.release();
    c->vroll_first.release(); c->vroll_state.release();
    c->vnext_row.release(); c->vrrec.release(); c->vlive.release();
    c->stats.release();
    delete c;
}

bs_status bs_sync_status(bs_ctx* c, void* stream, uint32_t* word) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    uint32_t w = 0;
    CK(c, cudaMemcpyAsync(&w, c->dev_err.p, sizeof w, cudaMemcpyDeviceToHost, S(stream)), "read error word");
    CK(c, cudaMemsetAsync(c->dev_err.p, 0, sizeof(uint32_t), S(stream)), "clear error word");
    CK(c, cudaStreamSynchronize(S(stream)), "bs_sync_status");
    if (word) *word = w;
    if (w & BS_DEV_STALE) return fail(c, BS_ERR_STALE, "device error word 0x%x: lookup against a stale index", w);
    if (w) return fail(c, BS_ERR_DEVICE, "device error word 0x%x", w);
    return BS_OK;
}

bs_status bs_rollout_begin(bs_ctx* c, int32_t n, const int32_t* slots, const uint64_t* uids,
                           const int32_t* prompt_ids, const int32_t* prompt_tail,
                           const int32_t* max_len, void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (n < 0 || n > c->cfg.max_rollouts) return fail(c, BS_ERR_INVALID, "n out of range");
    if (n && (!slots || !uids || !prompt_ids || !prompt_tail || !max_len))
        return fail(c, BS_ERR_INVALID, "null array");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    CK(c, launch_begin(c, n, slots, reinterpret_cast<const unsigned long long*>(uids), prompt_ids,
                       prompt_tail, max_len, S(stream)),
       "bs_rollout_begin");
    return BS_OK;
}

bs_status bs_rollout_state(bs_ctx* c, int32_t n, const int32_t* slots, int32_t* pos,
                           int32_t* finished, void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (n < 0 || n > c->cfg.max_rollouts) return fail(c, BS_ERR_INVALID, "n out of range");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    CK(c, launch_state(c, n, slots, pos, finished, S(stream)), "bs_rollout_state");
    return BS_OK;
}

bs_status bs_rollout_live(bs_ctx* c, int32_t n, const int32_t* slots, int32_t* live, void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (n < 0 || n > c->cfg.max_rollouts || !live || (n && !slots)) return fail(c, BS_ERR_INVALID, "bad arguments");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    CK(c, launch_live_count(c, n, slots, live, S(stream)), "bs_rollout_live");
    return BS_OK;
}

bs_status bs_draft_pool_put(bs_ctx* c, uint64_t rl_step, int32_t n_seqs, const int32_t* prompt_ids,
                            const int64_t* seq_offsets, const int32_t* tokens, int64_t n_tokens,
                            void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (n_seqs < 0 || n_tokens < 0) return fail(c, BS_ERR_INVALID, "negative size");
    if (n_seqs && (!prompt_ids || !seq_offsets)) return fail(c, BS_ERR_INVALID, "null array");
    if (n_tokens && !tokens) return fail(c, BS_ERR_INVALID, "null tokens");
    Pool& P = c->staging;
    if (!P.valid || P.step != rl_step) {
        P.valid = true;
        P.step = rl_step;
        P.n_tokens = 0;
        P.n_seqs = 0;
        bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
        // from here until the seal of rl_step, lookups of the older index are stale
        CK(c, bs::set_cur_step(c, rl_step, S(stream)), "bs_draft_pool_put");
    }
    if (P.n_tokens + n_tokens > c->cfg.pool_capacity_tokens ||
        (int64_t)P.n_seqs + n_seqs > c->cfg.pool_capacity_seqs)
        return fail(c, BS_ERR_CAPACITY, "pool capacity exceeded (%lld tokens, %d seqs)",
                    (long long)(P.n_tokens + n_tokens), P.n_seqs + n_seqs);
    if (n_seqs == 0) return BS_OK;
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    CK(c, launch_pool_append(c, n_seqs, prompt_ids, seq_offsets, tokens, n_tokens, S(stream)),
       "bs_draft_pool_put");
    P.n_tokens += n_tokens;
    P.n_seqs += n_seqs;
    return BS_OK;
}

bs_status bs_draft_pool_seal(bs_ctx* c, uint64_t rl_step, void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    Pool& P = c->staging;
    if (!P.valid || P.step != rl_step) {
        // a repeated seal of the step already sealed is a no-op (it must not seal an empty pool)
        if (c->sealed.valid && c->sealed.step == rl_step) return BS_OK;
        // nothing put for this step: an empty pool
        P.valid = true;
        P.step = rl_step;
        P.n_tokens = 0;
        P.n_seqs = 0;
        CK(c, cudaMemsetAsync(P.seq_off.p, 0, sizeof(int64_t), S(stream)), "seal");
    }
    // the index is built from the assembled pool; on failure the pools are swapped back, so the
    // assembled pool stays staged for a retry, and the index is published as invalid (its
    // lookups are stale) instead of leaving a half-built table in use
    std::swap(c->staging, c->sealed);
    c->sealed.step = rl_step;
    std::string why;
    cudaError_t e = seal_index(c, S(stream), why);
    if (e == cudaSuccess) e = bs::set_cur_step(c, rl_step, S(stream));
    if (e != cudaSuccess) {
        std::swap(c->staging, c->sealed);
        c->staging.valid = true;
        c->sealed.valid = false;
        bs::invalidate_index(c, S(stream));
        if (!why.empty()) return fail(c, BS_ERR_CAPACITY, "seal: %s", why.c_str());
        return cuda_fail(c, e, "bs_draft_pool_seal");
    }
    c->sealed.valid = true;
    c->staging.valid = false;
    return BS_OK;
}

bs_status bs_draft_lookup(bs_ctx* c, uint64_t rl_step, int32_t n, const int32_t* slots, int32_t k,
                          int32_t* draft_tokens, int32_t* draft_len, int32_t* match_len,
                          void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (!c->sealed.valid || c->sealed.step != rl_step)
        return fail(c, BS_ERR_STALE, "index not sealed for rl_step %llu", (unsigned long long)rl_step);
    if (n < 0 || n > c->cfg.max_rollouts) return fail(c, BS_ERR_INVALID, "n out of range");
    if (k < 0 || k > c->cfg.k_max) return fail(c, BS_ERR_INVALID, "k out of range");
    if (n && (!slots || !draft_len || (k && !draft_tokens))) return fail(c, BS_ERR_INVALID, "null array");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    CK(c, launch_lookup(c, n, slots, k, draft_tokens, draft_len, match_len, S(stream)),
       "bs_draft_lookup");
    return BS_OK;
}

bs_status bs_draft_set_min_token_prob(bs_ctx* c, float min_token_prob) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (!(min_token_prob >= 0.f && min_token_prob <= 1.f))
        return fail(c, BS_ERR_INVALID, "min_token_prob must be in [0, 1]");
    // reading C1: the threshold as round(tau * 2^32) in [0, 2^32], used by the next seal
    c->tau_q = (uint64_t)llround((double)min_token_prob * 4294967296.0);
    return BS_OK;
}

bs_status bs_draft_lookup_ngram(bs_ctx* c, uint64_t rl_step, int32_t n, const int32_t* slots, int32_t k,
                                int32_t n_min, int32_t n_max, int32_t* draft_tokens, int32_t* draft_len,
                                int32_t* match_len, void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (!c->sealed.valid || c->sealed.step != rl_step)
        return fail(c, BS_ERR_STALE, "index not sealed for rl_step %llu", (unsigned long long)rl_step);
    if (n < 0 || n > c->cfg.max_rollouts) return fail(c, BS_ERR_INVALID, "n out of range");
    if (k < 0 || k > c->cfg.k_max) return fail(c, BS_ERR_INVALID, "k out of range");
    if (n_min < 1 || n_max < n_min || n_max > c->M)
        return fail(c, BS_ERR_INVALID, "need 1 <= n_min <= n_max <= match_max");
    if (n && (!slots || !draft_len || (k && !draft_tokens))) return fail(c, BS_ERR_INVALID, "null array");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    CK(c, launch_lookup_ngram(c, n, slots, k, n_min, n_max, draft_tokens, draft_len, match_len, S(stream)),
       "bs_draft_lookup_ngram");
    return BS_OK;
}

// Host-side check of bs_sampling (returns the reason, or nullptr if valid).
static const char* sampling_invalid(const bs_sampling& sp) {
    if (!(sp.temperature >= 0.f) || sp.temperature == INFINITY) return "temperature must be finite and >= 0";
    if (!(sp.top_p > 0.f && sp.top_p <= 1.f)) return "top_p must be in (0, 1]";
    if (sp.top_k < 0) return "top_k must be >= 0";
    if (sp.temperature > 0.f && !((float)(1.4426950408889634 / (double)sp.temperature) < INFINITY))
        return "temperature too small";
    return nullptr;
}

bs_status bs_verify_step(bs_ctx* c, int32_t n, const int32_t* slots, const void* logits,
                         const int64_t* row_index, int64_t stride, const int32_t* draft_tokens,
                         const int32_t* draft_len, int32_t k, bs_sampling sp,
                         int32_t* out_tokens, int32_t* out_len, int32_t* out_accepted,
                         float* out_norm, uint64_t* out_z, void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (n < 0 || n > c->cfg.max_rollouts) return fail(c, BS_ERR_INVALID, "n out of range");
    if (k < 0 || k > c->cfg.k_max) return fail(c, BS_ERR_INVALID, "k out of range");
    if (stride < c->cfg.vocab) return fail(c, BS_ERR_INVALID, "row stride < vocab");
    if (const char* why = sampling_invalid(sp)) return fail(c, BS_ERR_INVALID, "%s", why);
    if (n && (!slots || !logits || !draft_len || !out_tokens || !out_len || !out_accepted ||
              (k && !draft_tokens)))
        return fail(c, BS_ERR_INVALID, "null array");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    CK(c, launch_verify(c, n, slots, logits, row_index, stride, draft_tokens, draft_len, k,
                        sp.temperature, sp.top_p, sp.top_k, out_tokens, out_len, out_accepted, out_norm,
                        reinterpret_cast<unsigned long long*>(out_z), S(stream)),
       "bs_verify_step");
    return BS_OK;
}

bs_status bs_verify_commit(bs_ctx* c, int32_t n, const int32_t* slots, const void* logits,
                           const int64_t* row_index, int64_t stride, const int32_t* draft_tokens,
                           const int32_t* draft_len, int32_t k, bs_sampling sp, int32_t* out_tokens,
                           int32_t* out_len, int32_t* out_accepted, float* out_norm, uint64_t* out_z,
                           int32_t* finished, void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (n < 0 || n > c->cfg.max_rollouts) return fail(c, BS_ERR_INVALID, "n out of range");
    if (k < 0 || k > c->cfg.k_max) return fail(c, BS_ERR_INVALID, "k out of range");
    if (stride < c->cfg.vocab) return fail(c, BS_ERR_INVALID, "row stride < vocab");
    if (const char* why = sampling_invalid(sp)) return fail(c, BS_ERR_INVALID, "%s", why);
    if (n && (!slots || !logits || !draft_len || !out_tokens || !out_len || !out_accepted ||
              (k && !draft_tokens)))
        return fail(c, BS_ERR_INVALID, "null array");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    bool fused = false;
    CK(c, launch_verify(c, n, slots, logits, row_index, stride, draft_tokens, draft_len, k,
                        sp.temperature, sp.top_p, sp.top_k, out_tokens, out_len, out_accepted, out_norm,
                        reinterpret_cast<unsigned long long*>(out_z), S(stream), finished, &fused),
       "bs_verify_commit");
    if (!fused)  // kernels without the fused commit: the commit kernel follows
        CK(c, launch_commit(c, n, slots, out_tokens, out_len, k, finished, S(stream)), "bs_verify_commit");
    return BS_OK;
}

bs_status bs_verify_commit_lookup(bs_ctx* c, uint64_t rl_step, int32_t n, const int32_t* slots,
                                  const void* logits, const int64_t* row_index, int64_t stride,
                                  int32_t* draft_tokens, int32_t* draft_len, int32_t k, bs_sampling sp,
                                  int32_t* out_tokens, int32_t* out_len, int32_t* out_accepted,
                                  float* out_norm, uint64_t* out_z, int32_t* finished, int32_t* match_len,
                                  void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (!c->sealed.valid || c->sealed.step != rl_step)
        return fail(c, BS_ERR_STALE, "index not sealed for rl_step %llu", (unsigned long long)rl_step);
    if (n < 0 || n > c->cfg.max_rollouts) return fail(c, BS_ERR_INVALID, "n out of range");
    if (k < 0 || k > c->cfg.k_max) return fail(c, BS_ERR_INVALID, "k out of range");
    if (stride < c->cfg.vocab) return fail(c, BS_ERR_INVALID, "row stride < vocab");
    if (const char* why = sampling_invalid(sp)) return fail(c, BS_ERR_INVALID, "%s", why);
    if (n && (!slots || !logits || !draft_len || !out_tokens || !out_len || !out_accepted ||
              (k && !draft_tokens)))
        return fail(c, BS_ERR_INVALID, "null array");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    bool fused = false, looked = false;
    const LookupArgs lk = lookup_args(c, n, slots, k, draft_tokens, draft_len, match_len);
    CK(c, launch_verify(c, n, slots, logits, row_index, stride, draft_tokens, draft_len, k,
                        sp.temperature, sp.top_p, sp.top_k, out_tokens, out_len, out_accepted, out_norm,
                        reinterpret_cast<unsigned long long*>(out_z), S(stream), finished, &fused, &lk,
                        &looked),
       "bs_verify_commit_lookup");
    if (!fused)
        CK(c, launch_commit(c, n, slots, out_tokens, out_len, k, finished, S(stream)), "bs_verify_commit_lookup");
    if (!looked)
        CK(c, launch_lookup(c, n, slots, k, draft_tokens, draft_len, match_len, S(stream)),
           "bs_verify_commit_lookup");
    return BS_OK;
}

bs_status bs_commit(bs_ctx* c, int32_t n, const int32_t* slots, const int32_t* out_tokens,
                    const int32_t* out_len, int32_t k, int32_t* finished, void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (n < 0 || n > c->cfg.max_rollouts) return fail(c, BS_ERR_INVALID, "n out of range");
    if (k < 0 || k > c->cfg.k_max) return fail(c, BS_ERR_INVALID, "k out of range");
    if (n && (!slots || !out_tokens || !out_len)) return fail(c, BS_ERR_INVALID, "null array");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    CK(c, launch_commit(c, n, slots, out_tokens, out_len, k, finished, S(stream)), "bs_commit");
    return BS_OK;
}

bs_status bs_stats_read(bs_ctx* c, uint64_t* out, int32_t n, int32_t reset, void* stream) {
    if (!c || (n && !out) || n < 0) return fail(c, BS_ERR_INVALID, "bad arguments");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    const int m = n < (int)STAT_COUNT ? n : (int)STAT_COUNT;
    if (m) CK(c, cudaMemcpyAsync(out, c->stats.p, m * sizeof(uint64_t), cudaMemcpyDeviceToHost, S(stream)), "stats");
    if (reset) CK(c, cudaMemsetAsync(c->stats.p, 0, STAT_COUNT * sizeof(uint64_t), S(stream)), "stats");
    CK(c, cudaStreamSynchronize(S(stream)), "stats");
    return BS_OK;
}

bs_status bs_rollout_bind_output(bs_ctx* c, int32_t* responses, int64_t stride) {
    if (!c || stride < 0 || (responses && stride == 0)) return fail(c, BS_ERR_INVALID, "bad arguments");
    c->responses = responses;
    c->resp_stride = responses ? stride : 0;
    return BS_OK;
}

bs_status bsx_synth_bank(void* bank, int64_t rows, int32_t V, uint32_t seed, float beta,
                         void* stream) {
    if (!bank || rows < 0 || V < 1) return fail(nullptr, BS_ERR_INVALID, "bad bank arguments");
    cudaError_t e = launch_synth_bank(bank, rows, V, seed, beta, S(stream));
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "bsx_synth_bank");
    return BS_OK;
}

bs_status bsx_target_rows(bs_ctx* c, int32_t n, const int32_t* slots, const int32_t* draft,
                          const int32_t* draft_len, int32_t k, uint32_t tseed, int32_t mode,
                          int64_t nbank, int64_t* row_index, void* stream) {
    if (!c) return fail(nullptr, BS_ERR_INVALID, "null ctx");
    if (n < 0 || n > c->cfg.max_rollouts || k < 0 || k > c->cfg.k_max || nbank < 1 || mode < 0 ||
        mode > 3 || (mode == 3 && nbank < 16))
        return fail(c, BS_ERR_INVALID, "bad target arguments");
    bs::DeviceScope dev_scope_(c->cfg.device);
    CK(c, dev_scope_.err, "cudaSetDevice");
    CK(c, launch_target_rows(c, n, slots, draft, draft_len, k, tseed, mode, nbank, row_index,
                             S(stream)),
       "bsx_target_rows");
    return BS_OK;
}

}  // extern "C"
