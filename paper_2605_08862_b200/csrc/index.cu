// index.cu — draft pool index build (K2, per RL step) and batched lookup (K1, per step).
//
// Lookup semantics (readings L1-L6):
//   anchor m* = longest suffix (<= M) of the rollout context that occurs in the prompt's
//   pool followed by a token; draft = greedy descent by occurrence count (ties -> lowest
//   id) for up to K tokens.
//
// Build (exact, no hashing): level l = 1..M+K sorts the active window occurrences by
// (run id of the length-(l-1) prefix, last token) with a device radix sort, so runs at
// level l are exactly the distinct windows of length l.  Unique windows drop out (their
// extensions are unique).  A descending pass computes, per distinct non-unique window,
// the end point of its greedy path (best child = largest child run, lowest token on ties;
// a unique child continues as plain text).  Windows of length <= M are inserted into a
// hashed table keyed (prompt, length, polynomial hash): every non-unique window, plus the
// FIRST unique window at each end position (its left extensions share its one occurrence
// and thus its draft).  The set of stored suffix lengths of any context is then contiguous,
// so lookup is one round of parallel probes (one lane per length) + one pool read.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "lookup.cuh"

namespace bs {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint64_t hash_window(const int32_t* T, int64_t start, int len) {
    uint64_t H = 0;
    for (int t = 0; t < len; ++t) H = H * HASH_B + (uint64_t)(uint32_t)(T[start + t] + 1);
    return H;
}

__device__ void table_insert(IndexEntry* table, uint64_t mask, uint64_t key, uint32_t occ,
                             uint32_t meta, uint32_t* dev_err) {
    uint64_t s = key & mask;
    for (;;) {
        unsigned long long prev = atomicCAS(&table[s].key, 0ull, (unsigned long long)key);
        if (prev == 0ull) {
            table[s].occ = occ;
            table[s].meta = meta;
            return;
        }
        if (prev == key) {  // two distinct windows with one 64-bit key
            atomicOr(dev_err, DEV_INDEX_KEY);
            return;
        }
        s = (s + 1) & mask;
    }
}

__global__ void seq_meta_kernel(const int64_t* seq_off, const int32_t* seq_prompt, int n_seqs,
                                int32_t* seq_start_of, int32_t* seq_end_of, int32_t* prompt_of) {
    for (int s = blockIdx.x; s < n_seqs; s += gridDim.x) {
        const int64_t a = seq_off[s], b = seq_off[s + 1];
        const int32_t P = seq_prompt[s];
        for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
            seq_start_of[i] = (int32_t)a;
            seq_end_of[i] = (int32_t)b;
            prompt_of[i] = P;
        }
    }
}

__global__ void iota_kernel(int32_t* a, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

__global__ void fill_kernel(int32_t* a, int n, int32_t v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = v;
}

__global__ void level_keys_kernel(int l, int A, int VB, const int32_t* act, const int32_t* T,
                                  const int32_t* prompt_of, const int32_t* runid_pos,
                                  unsigned long long* keys) {
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < A; a += gridDim.x * blockDim.x) {
        const int i = act[a];
        const uint64_t hi = (l == 1) ? (uint64_t)(uint32_t)prompt_of[i] : (uint64_t)(uint32_t)runid_pos[i];
        keys[a] = (hi << VB) | (uint64_t)(uint32_t)T[i + l - 1];
    }
}

__global__ void run_flags_kernel(int A, const unsigned long long* keys, int32_t* flag) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < A; r += gridDim.x * blockDim.x)
        flag[r] = (r == 0 || keys[r] != keys[r - 1]) ? 1 : 0;
}

__global__ void run_starts_kernel(int l, int A, int VB, const unsigned long long* keys,
                                  const int32_t* flag, const int32_t* runid_incl, int32_t* runstart,
                                  int32_t* parent) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < A; r += gridDim.x * blockDim.x) {
        if (flag[r]) {
            const int R = runid_incl[r] - 1;
            runstart[R] = r;
            parent[R] = (l == 1) ? -1 : (int32_t)(keys[r] >> VB);
        }
        if (r == A - 1) runstart[runid_incl[r]] = A;
    }
}

// per sorted element: record run id per position, first-unique level, next-level activity
__global__ void run_members_kernel(int l, int A, const int32_t* pos_sorted, const int32_t* runid_incl,
                                   const int32_t* runstart, const int32_t* seq_end_of,
                                   int32_t* runid_pos, int32_t* fu, int32_t* next_flag) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < A; r += gridDim.x * blockDim.x) {
        const int R = runid_incl[r] - 1;
        const int size = runstart[R + 1] - runstart[R];
        const int i = pos_sorted[r];
        runid_pos[i] = R;
        if (size == 1) {
            fu[i] = l;
            next_flag[r] = 0;
        } else {
            next_flag[r] = (i + l < seq_end_of[i]) ? 1 : 0;
        }
    }
}

struct Level {
    int A = 0, nruns = 0;
    int32_t* pos_sorted = nullptr;  // [A]
    int32_t* runstart = nullptr;    // [nruns + 1]
    int32_t* parent = nullptr;      // [nruns]
};

__global__ void child_ranges_kernel(int nruns_child, const int32_t* parent, int32_t* cbeg,
                                    int32_t* cend) {
    for (int C = blockIdx.x * blockDim.x + threadIdx.x; C < nruns_child; C += gridDim.x * blockDim.x) {
        const int p = parent[C];
        if (C == 0 || parent[C - 1] != p) cbeg[p] = C;
        if (C == nruns_child - 1 || parent[C + 1] != p) cend[p] = C + 1;
    }
}

// Descending pass at level l: greedy path end points for non-unique runs, table inserts
// for l <= M (non-unique windows, and first-unique windows).
__global__ void level_paths_kernel(int l, int M, int K, uint64_t tau_q, int top, Level lv, Level ch,
                                   const int32_t* cbeg, const int32_t* cend, const int32_t* pq_child,
                                   const int32_t* po_child, int32_t* pq, int32_t* po,
                                   const int32_t* T, const int32_t* seq_end_of,
                                   const int32_t* prompt_of, const int32_t* fu, IndexEntry* table,
                                   uint64_t mask, uint32_t* dev_err) {
    for (int R = blockIdx.x * blockDim.x + threadIdx.x; R < lv.nruns; R += gridDim.x * blockDim.x) {
        const int rs = lv.runstart[R];
        const int size = lv.runstart[R + 1] - rs;
        const int i0 = lv.pos_sorted[rs];
        if (size == 1) continue;  // unique windows: first_unique_kernel
        int q = 0, occ = i0;
        bool cont = false;  // the window has a continuation (anchor eligibility, L2)
        if (!top) {
            const int c0 = cbeg[R], c1 = cend[R];
            int best = -1, bsz = 0;
            for (int C = c0; C < c1; ++C) {  // children ordered by next token ascending
                const int sz = ch.runstart[C + 1] - ch.runstart[C];
                if (sz > bsz) {
                    bsz = sz;
                    best = C;
                }
            }
            cont = best >= 0;
            // reading C1: the greedy child's empirical probability bsz / size below tau ends the
            // draft here (q = 0); a child that passes continues with ITS (already gated) draft
            if (cont && ((uint64_t)bsz << 32) >= tau_q * (uint64_t)size) {
                const int cpos = ch.pos_sorted[ch.runstart[best]];
                if (bsz == 1) {
                    occ = cpos;
                    q = min(K, seq_end_of[cpos] - cpos - l);
                } else {
                    q = min(K, 1 + pq_child[best]);
                    occ = po_child[best];
                }
            }
        }
        pq[R] = q;
        po[R] = occ;
        if (l <= M) {
            const uint32_t meta = (uint32_t)q | (cont ? META_CONT : 0u);
            table_insert(table, mask, window_key(hash_window(T, occ, l), prompt_of[occ], l),
                         (uint32_t)occ, meta, dev_err);
        }
    }
}

// First-unique windows.  fu[i] = the length at which the window starting at i became
// unique (its extensions stay unique and share its single occurrence).  The window (i, l)
// is the FIRST unique window at its end position e = i+l-1 iff it is unique (l >= fu[i])
// and (i+1, l-1) is not (l <= fu[i+1]); so position i contributes the lengths
// [fu[i], min(fu[i+1], M, seq_end - i)].  At most one entry per end position.
__global__ void first_unique_kernel(int n, int M, int K, const int32_t* T, const int32_t* fu,
                                    const int32_t* seq_end_of, const int32_t* prompt_of,
                                    IndexEntry* table, uint64_t mask, uint32_t* dev_err) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int lo = fu[i];
        if (lo > M) continue;
        const int se = seq_end_of[i];
        int hi = min(M, se - i);
        if (i + 1 < se) hi = min(hi, fu[i + 1]);
        if (lo > hi) continue;
        const int32_t P = prompt_of[i];
        uint64_t H = 0;
        for (int t = 0; t < lo - 1; ++t) H = H * HASH_B + (uint64_t)(uint32_t)(T[i + t] + 1);
        for (int l = lo; l <= hi; ++l) {
            H = H * HASH_B + (uint64_t)(uint32_t)(T[i + l - 1] + 1);
            const int q = min(K, se - (i + l));
            const uint32_t meta = (uint32_t)q | META_UNIQUE | (q > 0 ? META_CONT : 0u);
            table_insert(table, mask, window_key(H, P, l), (uint32_t)i, meta, dev_err);
        }
    }
}

static int bits_for(uint64_t v) {
    int b = 0;
    while (b < 64 && (v >> b) != 0) ++b;
    return b;
}

#define BS_TRY(x)                       \
    do {                                \
        cudaError_t e__ = (x);          \
        if (e__ != cudaSuccess) return e__; \
    } while (0)

// The lookup kernel reads the sealed index through a device-resident descriptor, so a
// captured decode-step graph stays valid when a later seal reallocates the index.
static cudaError_t publish_index(bs_ctx* ctx, cudaStream_t st, unsigned long long step) {
    IndexDesc d;
    d.step = step;
    d.table = ctx->table.p;
    d.mask = ctx->table_mask;
    d.T = ctx->sealed.tokens.p;
    d.seq_start_of = ctx->seq_start_of.p;
    d.seq_off = ctx->sealed.seq_off.p;
    d.seq_prompt = ctx->sealed.seq_prompt.p;
    d.n_seqs = ctx->sealed.n_seqs;
    return cudaMemcpyAsync(ctx->idx_desc.p, &d, sizeof d, cudaMemcpyHostToDevice, st);  // pageable: staged now
}

cudaError_t set_cur_step(bs_ctx* ctx, uint64_t step, cudaStream_t st) {
    const unsigned long long v = step;
    return cudaMemcpyAsync(ctx->cur_step.p, &v, sizeof v, cudaMemcpyHostToDevice, st);  // pageable: staged now
}

void invalidate_index(bs_ctx* ctx, cudaStream_t st) {
    publish_index(ctx, st, ~0ull);
    cudaStreamSynchronize(st);
}

cudaError_t seal_index(bs_ctx* ctx, cudaStream_t st, std::string& why) {
    const int64_t N = ctx->sealed.n_tokens;
    const int M = ctx->M, K = ctx->cfg.k_max, D = M + K;
    const int V = ctx->cfg.vocab;
    const int VB = std::max(1, bits_for((uint64_t)V));
    if (N >= (int64_t)0x7FFFFFFF) {
        why = "pool too large for 32-bit positions";
        return cudaErrorInvalidValue;
    }
    const int n = (int)N;
    BS_TRY(ctx->seq_start_of.ensure_async(n, st));
    BS_TRY(ctx->seq_end_of.ensure_async(n, st));
    BS_TRY(ctx->prompt_of.ensure_async(n, st));
    if (ctx->sealed.n_seqs > 0 && n > 0)
        seq_meta_kernel<<<std::min(ctx->sealed.n_seqs, 4096), 256, 0, st>>>(
            ctx->sealed.seq_off.p, ctx->sealed.seq_prompt.p, ctx->sealed.n_seqs, ctx->seq_start_of.p,
            ctx->seq_end_of.p, ctx->prompt_of.p);
    if (n == 0) {
        BS_TRY(ctx->table.ensure_async(2, st));
        BS_TRY(cudaMemsetAsync(ctx->table.p, 0, 2 * sizeof(IndexEntry), st));
        ctx->table_mask = 1;
        BS_TRY(publish_index(ctx, st, ctx->sealed.step));
        return cudaStreamSynchronize(st);
    }
    const int* T = ctx->sealed.tokens.p;
    // scratch (stream-ordered: no synchronising cudaMalloc / cudaFree per seal)
    AsyncBuf<int32_t> act, act_next, flag, runid, runid_pos, fu, nflag;
    AsyncBuf<unsigned long long> keys, keys_sorted;
    AsyncBuf<int> d_count;
    BS_TRY(act.alloc(n, st));
    BS_TRY(act_next.alloc(n, st));
    BS_TRY(flag.alloc(n, st));
    BS_TRY(runid.alloc(n, st));
    BS_TRY(runid_pos.alloc(n, st));
    BS_TRY(fu.alloc(n, st));
    BS_TRY(nflag.alloc(n, st));
    BS_TRY(keys.alloc(n, st));
    BS_TRY(keys_sorted.alloc(n, st));
    BS_TRY(d_count.alloc(1, st));
    size_t tmp_bytes = 0, t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, keys.p, keys_sorted.p, act.p, act_next.p, n, 0, 64, st);
    cub::DeviceScan::InclusiveSum(nullptr, t2, flag.p, runid.p, n, st);
    cub::DeviceSelect::Flagged(nullptr, t3, act.p, nflag.p, act_next.p, d_count.p, n, st);
    tmp_bytes = std::max(t1, std::max(t2, t3));
    AsyncBuf<uint8_t> tmp;
    BS_TRY(tmp.alloc(tmp_bytes, st));
    const int G = std::max(1, std::min(ctx->num_sms * 8, (n + 255) / 256));
    iota_kernel<<<G, 256, 0, st>>>(act.p, n);
    fill_kernel<<<G, 256, 0, st>>>(fu.p, n, 0x7FFFFFFF);

    std::vector<Level> levels;
    struct LevelFree {  // per-level arrays: stream-ordered frees on every exit path
        std::vector<Level>& lv;
        cudaStream_t st;
        ~LevelFree() {
            for (auto& l : lv) {
                if (l.pos_sorted) cudaFreeAsync(l.pos_sorted, st);
                if (l.runstart) cudaFreeAsync(l.runstart, st);
                if (l.parent) cudaFreeAsync(l.parent, st);
            }
        }
    } level_free{levels, st};
    int A = n;
    uint64_t hi_max = 0;  // max of the high key part (prompt id or previous run count)
    {
        // prompt ids are int32: use the full 32 bits at level 1
        hi_max = 0xFFFFFFFFull;
    }
    for (int l = 1; l <= D && A > 0; ++l) {
        levels.push_back(Level{});
        Level& lv = levels.back();
        lv.A = A;
        BS_TRY(cudaMallocAsync(reinterpret_cast<void**>(&lv.pos_sorted), sizeof(int32_t) * (size_t)A, st));
        const int g = std::max(1, std::min(ctx->num_sms * 8, (A + 255) / 256));
        level_keys_kernel<<<g, 256, 0, st>>>(l, A, VB, act.p, T, ctx->prompt_of.p, runid_pos.p, keys.p);
        const int end_bit = std::min(64, VB + bits_for(hi_max));
        size_t tb = tmp_bytes;
        BS_TRY(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.p, keys_sorted.p, act.p, lv.pos_sorted, A, 0,
                                               end_bit, st));
        run_flags_kernel<<<g, 256, 0, st>>>(A, keys_sorted.p, flag.p);
        tb = tmp_bytes;
        BS_TRY(cub::DeviceScan::InclusiveSum(tmp.p, tb, flag.p, runid.p, A, st));
        int nr = 0;
        BS_TRY(cudaMemcpyAsync(&nr, runid.p + (A - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
        BS_TRY(cudaStreamSynchronize(st));
        lv.nruns = nr;
        BS_TRY(cudaMallocAsync(reinterpret_cast<void**>(&lv.runstart), sizeof(int32_t) * (size_t)(nr + 1), st));
        BS_TRY(cudaMallocAsync(reinterpret_cast<void**>(&lv.parent), sizeof(int32_t) * (size_t)std::max(nr, 1), st));
        run_starts_kernel<<<g, 256, 0, st>>>(l, A, VB, keys_sorted.p, flag.p, runid.p, lv.runstart, lv.parent);
        run_members_kernel<<<g, 256, 0, st>>>(l, A, lv.pos_sorted, runid.p, lv.runstart, ctx->seq_end_of.p,
                                              runid_pos.p, fu.p, nflag.p);
        tb = tmp_bytes;
        BS_TRY(cub::DeviceSelect::Flagged(tmp.p, tb, lv.pos_sorted, nflag.p, act.p, d_count.p, A, st));
        int an = 0;
        BS_TRY(cudaMemcpyAsync(&an, d_count.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        BS_TRY(cudaStreamSynchronize(st));
        A = an;
        hi_max = (uint64_t)nr;
    }
    // table capacity: one entry per run at levels <= M, plus one first-unique per end position
    int64_t cap_need = n;
    for (size_t li = 0; li < levels.size() && (int)li < M; ++li) cap_need += levels[li].nruns;
    uint64_t cap = 2;
    while (cap < (uint64_t)(2 * cap_need + 2)) cap <<= 1;
    BS_TRY(ctx->table.ensure_async(cap, st));
    BS_TRY(cudaMemsetAsync(ctx->table.p, 0, cap * sizeof(IndexEntry), st));
    ctx->table_mask = cap - 1;
    first_unique_kernel<<<G, 256, 0, st>>>(n, M, K, T, fu.p, ctx->seq_end_of.p, ctx->prompt_of.p,
                                           ctx->table.p, ctx->table_mask, ctx->dev_err.p);
    // descending pass
    int maxr = 1;
    for (auto& lv : levels) maxr = std::max(maxr, lv.nruns);
    AsyncBuf<int32_t> pqa, poa, pqb, pob, cbeg, cend;
    BS_TRY(pqa.alloc(maxr, st));
    BS_TRY(poa.alloc(maxr, st));
    BS_TRY(pqb.alloc(maxr, st));
    BS_TRY(pob.alloc(maxr, st));
    BS_TRY(cbeg.alloc(maxr, st));
    BS_TRY(cend.alloc(maxr, st));
    int32_t *pq_child = pqb.p, *po_child = pob.p, *pq = pqa.p, *po = poa.p;
    const int L = (int)levels.size();
    for (int li = L - 1; li >= 0; --li) {
        const int l = li + 1;
        Level lv = levels[li];
        Level ch;
        const int top = (li == L - 1) ? 1 : 0;
        if (!top) {
            ch = levels[li + 1];
            BS_TRY(cudaMemsetAsync(cbeg.p, 0, sizeof(int32_t) * (size_t)lv.nruns, st));
            BS_TRY(cudaMemsetAsync(cend.p, 0, sizeof(int32_t) * (size_t)lv.nruns, st));
            const int gc = std::max(1, std::min(ctx->num_sms * 8, (ch.nruns + 255) / 256));
            if (ch.nruns > 0) child_ranges_kernel<<<gc, 256, 0, st>>>(ch.nruns, ch.parent, cbeg.p, cend.p);
        }
        const int gr = std::max(1, std::min(ctx->num_sms * 8, (lv.nruns + 255) / 256));
        level_paths_kernel<<<gr, 256, 0, st>>>(l, M, K, ctx->tau_q, top, lv, ch, cbeg.p, cend.p, pq_child, po_child, pq, po,
                                               T, ctx->seq_end_of.p, ctx->prompt_of.p, fu.p, ctx->table.p,
                                               ctx->table_mask, ctx->dev_err.p);
        BS_TRY(cudaGetLastError());
        std::swap(pq, pq_child);
        std::swap(po, po_child);
    }
    BS_TRY(publish_index(ctx, st, ctx->sealed.step));
    return cudaStreamSynchronize(st);
}

// ------------------------------------------------------------------ lookup (K1)
__global__ void __launch_bounds__(256) lookup_kernel(const LookupArgs a) {
    pdl_wait();
    // dependents are triggered only after the drafts are stored (end of the kernel): the
    // verify kernel plans from them before its own griddepcontrol.wait
    const int lane = threadIdx.x & 31;
    const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= a.n) return;
    const IndexDesc x = *a.desc;
    const unsigned long long cur = *a.cur_step;
    const int slot = a.slots[b];
    const int M = a.M;
    // the slot's state and its whole tail go out together (one round trip)
    const int L = a.ctx_len[slot];
    const int P = a.prompt[slot];
    const int p = a.pos[slot], ml = a.max_len[slot];
    const int tok_raw = (lane < M) ? a.tail[(int64_t)slot * M + (M - 1 - lane)] : -1;  // y[-1-lane]
    const bool fin = a.finished[slot] != 0;
    lookup_rollout(a, x, b, L, P, p, ml, fin, tok_raw, lane, x.step != cur);
    __threadfence();
    pdl_trigger();
}

LookupArgs lookup_args(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t k, int32_t* draft,
                       int32_t* draft_len, int32_t* match_len) {
    LookupArgs a;
    a.slots = slots;
    a.n = n;
    a.k = k;
    a.M = ctx->M;
    a.Lmin = ctx->cfg.match_min;
    a.tail = ctx->tail.p;
    a.ctx_len = ctx->ctx_len.p;
    a.prompt = ctx->prompt.p;
    a.pos = ctx->pos.p;
    a.max_len = ctx->max_len.p;
    a.finished = ctx->finished.p;
    a.desc = ctx->idx_desc.p;
    a.cur_step = ctx->cur_step.p;
    a.dev_err = ctx->dev_err.p;
    a.draft = draft;
    a.draft_len = draft_len;
    a.match_len = match_len;
    return a;
}

cudaError_t launch_lookup(bs_ctx* ctx, int32_t n, const int32_t* slots, int32_t k, int32_t* draft,
                          int32_t* draft_len, int32_t* match_len, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const LookupArgs a = lookup_args(ctx, n, slots, k, draft, draft_len, match_len);
    const int blocks = (n * 32 + 255) / 256;
    cudaError_t le = launch_pdl(lookup_kernel, dim3(blocks), dim3(256), 0, st, a);
    if (le != cudaSuccess) return le;
    return cudaGetLastError();
}

}  // namespace bs
