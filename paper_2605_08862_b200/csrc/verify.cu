// verify.cu — fused vocab-row verify + resample (Eq. 2, Eq. 3 P:208-210,
// Alg. 1, bonus token P:308) for sm_100a.
//
// Kernel K3.  One persistent CTA per SM verifies whole logits rows with no
// cross-CTA synchronisation, warp-specialized:
//   * PRODUCER warp: claims rows and streams each row twice through an 8-stage ring of
//     16 KB shared-memory chunks with 1-D bulk async copies (TMA engine, mbarrier
//     completion): pass 1 from HBM (left in L2), pass 2 re-read from L2 (evict-first);
//   * 16 CONSUMER warps: pass 1 = NaN-propagating bf16x2 row max (the only CTA barrier
//     of a row); pass 2 = integer masses of reading R (packed FFMA2/FADD2, exact u64
//     sums, one warp-level sum per 1024-element block) handed to the epilogue through a
//     double-buffered shared-memory record; then straight on to the next row;
//   * EPILOGUE warp: Z, mass(d), the accept test (Philox counter (pos+j, ACCEPT)) and,
//     when needed, the residual / bonus sample (inverse CDF: block sums locate the
//     crossing 1024-element block, the warp rescans it from L2), then the rollout's
//     bookkeeping — all off the consumers' critical path.
// Rows are claimed in Alg. 1's order across the batch — (b, 0) of every live rollout,
// then (b, 1), ... — and a row is SKIPPED when a lower row of its rollout already
// decided (first rejection / accepted EOS): rows after the first rejection are read only
// when they were claimed speculatively before that rejection was known.  Rows
// complete out of order; per rollout, atomicMin keeps the first deciding row and atomicOr
// the set of completed rows, and the row that completes the prefix finalizes (CAS).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cooperative_groups.h>

#include "common.cuh"
#include "ctx.h"
#include "ptx.cuh"
#include "verify_math.cuh"
#include "lookup.cuh"

namespace bs {

constexpr int CHE = 8192;           // elements per ring chunk (16 KB)
constexpr int NSTAGE = 4;           // ring depth (64 KB per CTA)
constexpr int NCW = 8;              // consumer warps
constexpr int CTAS_PER_SM = 2;      // one CTA's HBM pass overlaps the other's mass pass
constexpr int NCT = NCW * 32;       // consumer threads
constexpr int PROD_WARP = NCW;      // producer warp
constexpr int EPI_WARP = NCW + 1;   // epilogue warp
constexpr int NTHR = NCT + 64;
constexpr int RF = 4;               // row descriptor FIFO depth
constexpr int MAXG = 32;            // max super-chunks (2 chunks each): V <= 524288
constexpr int BLK = CHE * 2 / NCW;  // elements per warp per super-chunk (2048: 8 tiles)
constexpr int TPW = BLK / 256;      // 256-element tiles per warp per chunk
constexpr int EPL = BLK / 32;       // elements per lane when the epilogue rescans a block
// row status; ST_ERR: the row is invalid (reading R0), its candidate holds the error bits.  An
// error row decides like a rejection (Alg. 1 reads nothing above it) and is reported only if
// it is the rollout's deciding row, i.e. only if Alg. 1 needs it (the oracle stops there).
constexpr int ST_CONT = 0, ST_DECIDED = 1, ST_EOS = 2, ST_ERR = 3;
constexpr bool c_claim_early = false;  // producer claims row r+1 under row r's pass 1

// Optional per-stage cycle accounting (build with -DBS_PHASE_TIMING; read with
// bsx_phase_times): consumer thread 0 adds the clock64() delta of each phase.
#ifdef BS_PHASE_TIMING
__device__ unsigned long long g_phase[16];
#define PH_MARK(i)                                                     \
    do {                                                               \
        if (tid == 0) {                                                \
            const long long now_ = clock64();                          \
            atomicAdd(&g_phase[i], (unsigned long long)(now_ - ph_t)); \
            ph_t = now_;                                               \
        }                                                              \
    } while (0)
#else
#define PH_MARK(i) \
    do {           \
    } while (0)
#endif

struct RowDesc;

// Optional event trace (build with -DBS_TRACE; read with bsx_trace_read): globaltimer stamps
// of each row's stages per CTA, for latency analysis (scripts/trace_verify.py).
#ifdef BS_TRACE
// per-CTA slices of 2048 events; the index comes from a shared-memory counter (no global
// round trip), the store is fire-and-forget, so recording barely perturbs the timing
constexpr int TRACE_PER_CTA = 2048;
__device__ uint4 g_trace[1 << 20];
__device__ unsigned int g_trace_n;
__shared__ unsigned int s_trace_n;
__device__ __forceinline__ void trace_ev(int type, int seq, int b, int j) {
    const unsigned i = atomicAdd(&s_trace_n, 1u);
    const unsigned slot = blockIdx.x * TRACE_PER_CTA + i;
    if (i < TRACE_PER_CTA && slot < (1u << 20)) {
        const uint64_t t = globaltimer_ns();
        g_trace[slot] = make_uint4((uint32_t)blockIdx.x | ((uint32_t)type << 16) | ((uint32_t)(j & 0xFF) << 24),
                                   (uint32_t)(seq & 0xFFFF) | ((uint32_t)(b & 0xFFFF) << 16), (uint32_t)t,
                                   (uint32_t)(t >> 32));
    }
}
#define TRACE(type, seq, b, j) trace_ev(type, seq, b, j)
#else
#define TRACE(type, seq, b, j) \
    do {                       \
    } while (0)
#endif
enum { TR_CLAIM0 = 0, TR_CLAIM1 = 1, TR_TMA = 2, TR_MAX0 = 3, TR_MAX1 = 4, TR_MASS0 = 5, TR_MASS1 = 6,
       TR_EPI0 = 7, TR_EPI1 = 8, TR_END = 9, TR_FIN = 10, TR_SPINS = 11, TR_SC = 12, TR_SQPOP = 13, TR_ITER = 14, TR_MASSL = 15, TR_START = 16, TR_GO = 17, TR_PLANNED = 18, TR_PDESC = 19, TR_POST = 20, TR_LOOP = 21, TR_BCAST = 22, TR_EX1 = 24, TR_EX2 = 25, TR_EX3 = 26 };


struct VerifyArgs {
    const int32_t* slots;
    const uint16_t* logits;
    const int64_t* row_index;
    int64_t stride;
    const int32_t* draft;
    int32_t k, V, S, eos, nchunk, ngroup;
    float T, c;
    unsigned long long seed;
    const int32_t* pos;
    const unsigned long long* uid;
    const int32_t* rb_q;
    const RowDesc* items;  // the step's rows, j-major (plan kernel)
    unsigned int* ctl;            // VCTL_* words
    uint32_t* dev_err;
    int32_t* row_status;
    int32_t* row_cand;
    unsigned long long* row_z;
    float* row_norm;
    int32_t* roll_first;                 // lowest deciding row seen so far (claim hint)
    unsigned long long* roll_state;      // rows completed (bits 0-31) | rows deciding (32-63)
    int32_t* out_tokens;
    int32_t* out_len;
    int32_t* out_acc;
    float* out_norm;
    unsigned long long* out_z;
    unsigned long long* stats;
    // cluster-kernel scheduler (verify_cluster.cuh); sctl == nullptr for the other kernels
    int n;                        // rollouts of this call
    const int32_t* draft_len;
    const int32_t* max_len;
    const int32_t* finished;
    unsigned int* sctl;           // vctl words SC_*
    unsigned long long* next_row; // per rollout: epoch << 32 | next unclaimed row
    RollRec* rrec;                // per rollout: the launch's plan
    unsigned long long* live;     // live rollouts (epoch << 32 | b), compacted by the planners
    // fused commit (bs_verify_commit): the finalizing thread appends the rollout's tokens
    int commit, M;
    int32_t* c_tail;
    int32_t* c_ctx_len;
    int32_t* c_pos;
    int32_t* c_finished;
    int32_t* c_fin_out;
    int32_t* c_resp;
    int64_t c_resp_stride;
    int ncl;                      // clusters in the grid
    int eager_ok;                 // small live batches claim every row at once
    int early_plan;               // plan before griddepcontrol.wait (bsx_set_early_plan)
    // fused lookup (bs_verify_commit_lookup): after its commit, the finalizing warp looks up
    // the rollout's next draft from the committed state (lk.draft / draft_len: the next step's)
    int lookup;
    LookupArgs lk;
    // row statistics precomputed by the LM-head epilogue (bsx_set_row_stats; cluster kernel):
    // per logits row, (order key of the max << 32 | ~argmax) and a NaN / +inf flag
    const unsigned long long* rs_key;
    const uint32_t* rs_bad;
};

struct RowDesc {
    int32_t b, j, q, d;  // rollout, row, clamped draft length, d_{j+1} (-1 if j == q); b < 0: end
    int64_t rowno;       // logits row
    unsigned long long uid;  // rollout uid (Philox counter words 2-3, R6)
    int32_t position;    // generated-token index of the row's sample (Philox counter word 0)
    int32_t aligned;     // bulk copies usable (16-byte aligned row)
    int32_t pad[2];
};
static_assert(sizeof(RowDesc) == 48, "RowDesc layout");

// Philox draw for row dsc and purpose (R6): key = seed, counter = (position, purpose, uid).
__device__ __forceinline__ U128 row_draw(const VerifyArgs& a, const RowDesc& dsc, uint32_t purpose) {
    return draw(a.seed, dsc.uid, (uint32_t)dsc.position, purpose);
}

// Consumer -> epilogue handoff of one row (double-buffered).
struct EpiBuf {
    RowDesc dsc;
    float m;
    int32_t ok;
    uint32_t err;  // R0 error bits of the row (ok == 0)
    int32_t pad[1];
    unsigned long long csum[MAXG][NCW];  // exact sums of the 1024-element blocks (greedy:
                                         // csum[0][w] = first argmax index of warp w)
};

struct __align__(16) VShared {
    uint64_t full[NSTAGE];
    uint64_t empty[NSTAGE];
    uint64_t rfull[RF];
    uint64_t rempty[RF];
    uint64_t efull[2];
    uint64_t eempty[2];
    RowDesc desc[RF];
    float wmax[NCW];
    uint32_t wbad[NCW];
    EpiBuf epi[2];
    unsigned long long stat[STAT_COUNT];
};

// Alg. 1 lines 15/22 ("y <- y o a") for one rollout, by the warp whose lane 0 just
// finalized its step: the same state update as commit_kernel (state.cu), fused into the
// verify launch.  Lane i owns tail slot i (M <= 32) and emitted token i (<= k+1 <= 32).
struct CommitPre {
    int s, p, L, cl, old;  // slot, pos, max_len, ctx_len; lane i: tail slot i
    int P;                 // prompt (fused lookup)
    IndexDesc x;           // the sealed index (fused lookup)
    unsigned long long cur;  // rl_step of the latest put / seal (staleness)
};
__device__ __forceinline__ CommitPre commit_prefetch(const VerifyArgs& a, int slot, int lane) {
    CommitPre c;
    c.s = slot;
    c.p = a.c_pos[slot];
    c.L = a.max_len[slot];
    c.cl = a.c_ctx_len[slot];
    c.old = (lane < a.M) ? a.c_tail[(int64_t)slot * a.M + lane] : -1;
    if (a.lookup) {
        c.P = a.lk.prompt[slot];
        c.x = *a.lk.desc;
        c.cur = *a.lk.cur_step;
    }
    return c;
}

// The emitted block comes in registers from the warp's finalize: no (all lanes), lane i: token i.
__device__ void commit_rollout_warp(const VerifyArgs& a, int b, int lane, const CommitPre& c, int no, int32_t ot) {
    const int s = c.s;
    const int M = a.M;
    const int p = c.p, L = c.L;
    int32_t* tl = a.c_tail + (int64_t)s * M;
    const int32_t old = c.old;
    if (lane >= no) ot = -1;
    const int src = lane + no;  // new tail[i] = (old ++ out)[i + no]
    const int32_t from_old = __shfl_sync(0xFFFFFFFFu, old, src & 31);
    const int32_t from_out = __shfl_sync(0xFFFFFFFFu, ot, (src - M) & 31);
    const int32_t nt = (src < M) ? from_old : from_out;  // new tail[lane]
    if (lane < M) tl[lane] = nt;
    if (a.c_resp && lane < no && p + lane < a.c_resp_stride) a.c_resp[(int64_t)s * a.c_resp_stride + p + lane] = ot;
    const int32_t last = __shfl_sync(0xFFFFFFFFu, ot, (no - 1) & 31);
    // an empty block of a live rollout is an error stop (reading R0; as commit_kernel)
    const int f = (no == 0 || (a.eos >= 0 && last == a.eos) || p + no >= L) ? 1 : 0;
    if (lane == 0) {
        a.c_ctx_len[s] = min(M, c.cl + no);
        a.c_pos[s] = p + no;
        if (f) a.c_finished[s] = 1;
        if (a.c_fin_out) a.c_fin_out[b] = f;
    }
    if (a.lookup) {  // the next step's draft from the committed state: y[-1-lane] = tail[M-1-lane]
        const int32_t y = __shfl_sync(0xFFFFFFFFu, nt, (M - 1 - lane) & 31);
        lookup_rollout(a.lk, c.x, b, min(M, c.cl + no), c.P, p + no, L, f != 0, lane < M ? y : -1, lane,
                       c.x.step != c.cur);
    }
}

// Alg. 1 lines 10-31 for rollout b, decided at row F (rows < F accepted).
__device__ void finalize_rollout(const VerifyArgs& a, unsigned long long* s, int b, int F, int q) {
    const int kp1 = a.k + 1;
    int32_t* out = a.out_tokens + (int64_t)b * kp1;
    const int32_t* d = a.draft + (int64_t)b * a.k;
    const int64_t base = (int64_t)b * kp1;
    const int st = __ldcg(a.row_status + base + F);
    if (st == ST_ERR) {  // a needed row is invalid (R0): the step emits nothing, the error is reported
        atomicOr(a.dev_err, (uint32_t)__ldcg(a.row_cand + base + F));
        for (int i = 0; i < kp1; ++i) out[i] = -1;
        a.out_len[b] = 0;
        a.out_acc[b] = 0;
        if (a.sctl) atomicAdd(a.sctl + SC_DONE, 1u);
        return;
    }
    int n = 0;
    for (int i = 0; i < F; ++i) out[n++] = d[i];
    int acc = F;
    if (st == ST_EOS) {  // accepted EOS ends the block: no sample
        out[n++] = d[F];
        acc = F + 1;
    } else {
        out[n++] = __ldcg(a.row_cand + base + F);
    }
    for (int i = n; i < kp1; ++i) out[i] = -1;
    a.out_len[b] = n;
    a.out_acc[b] = acc;
    for (int i = 0; i <= F; ++i) {  // the rows Alg. 1 needed
        if (a.out_norm) a.out_norm[base + i] = __ldcg(a.row_norm + base + i);
        if (a.out_z) a.out_z[base + i] = __ldcg(a.row_z + base + i);
    }
    if (q > 0) {
        s[STAT_STEPS_SPEC] += 1ull;
        s[STAT_EMIT_SPEC] += (unsigned long long)n;
        s[STAT_ACCEPTED] += (unsigned long long)acc;
        s[STAT_PROPOSED] += (unsigned long long)q;
        s[STAT_HIST + min(n, STAT_HIST_BINS - 1)] += 1ull;
    } else {
        s[STAT_STEPS_PLAIN] += 1ull;
        s[STAT_EMIT_PLAIN] += (unsigned long long)n;
    }
    s[STAT_ROWS_NEEDED] += (unsigned long long)(F + 1);
    if (a.sctl) {
        const unsigned dn = atomicAdd(a.sctl + SC_DONE, 1u);  // scheduler termination count
        TRACE(TR_FIN, (int)dn, b, F);
    }
}

// Rollout state word: bit j = row j completed, bit 32+j = row j decides (reject / bonus /
// accepted EOS).  Alg. 1 is decided once the lowest deciding row F and every row below it
// are complete; that predicate only turns true once under OR, so the single atomic that
// makes it true finalizes (no CAS, no store-buffering hazard).
__device__ __forceinline__ bool prefix_decided(unsigned long long st, int& F) {
    const uint32_t dec = (uint32_t)(st >> 32);
    if (!dec) return false;
    F = __ffs(dec) - 1;
    const uint32_t need = (F >= 31) ? 0xFFFFFFFFu : ((2u << F) - 1u);
    return ((uint32_t)st & need) == need;
}

__device__ __forceinline__ unsigned long long atom_or_acq_rel(unsigned long long* p, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.or.b64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}

__device__ __forceinline__ unsigned long long atom_or_acquire(unsigned long long* p, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.acquire.gpu.global.or.b64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}

__device__ __forceinline__ void red_or_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Record a completed row and finalize its rollout if this completes the decided prefix.
// Returns true when this row's completion finalized the rollout's step.
__device__ bool complete_row(const VerifyArgs& a, unsigned long long* stat, int b, int j, int q, int status,
                             int cand, unsigned long long z, float norm) {
    const int64_t r = (int64_t)b * (a.k + 1) + j;
    a.row_status[r] = status;
    a.row_cand[r] = cand;
    a.row_z[r] = z;
    a.row_norm[r] = norm;
    const bool decides = status != ST_CONT;
    if (decides) atomicMin(a.roll_first + b, j);  // claim hint only (relaxed)
    const unsigned long long mine = (1ull << j) | (decides ? (1ull << (32 + j)) : 0ull);
    // release: this row's record; acquire: every earlier row's record of the rollout
    const unsigned long long old = atom_or_acq_rel(a.roll_state + b, mine);
    int F0, F1;
    if (!prefix_decided(old, F0) && prefix_decided(old | mine, F1)) {
        finalize_rollout(a, stat, b, F1, q);
        return true;
    }
    return false;
}

// complete_row for a whole warp (lane 0 records and ORs; on finalization the warp reads the
// decided prefix in one parallel round trip: lane i < F the draft token d_{i+1}, lane i <= F
// row i's normaliser / Z, the deciding row F's status and candidate; row j's own values come
// from registers).  Returns (all lanes) whether this row finalized the rollout's step; then
// no = emitted tokens and lane i holds emitted token i (inputs of the fused commit).
// dpf: lane i's draft token d_{i+1} (lane < q) if the caller prefetched it, else DPF_NONE.
constexpr int32_t DPF_NONE = -0x7FFFFFFF;
__device__ bool complete_row_warp(const VerifyArgs& a, unsigned long long* stat, int b, int j, int q, int status,
                                  int cand, unsigned long long z, float norm, int lane, int& no, int32_t& tok,
                                  int32_t dpf = DPF_NONE) {
    const int kp1 = a.k + 1;
    const int64_t base = (int64_t)b * kp1;
    int F = -1;
    const bool decides = status != ST_CONT;
    if (j == 0 && decides) {
        // Row 0 decides: F = 0 and this completion is the one that finalizes (rows are claimed
        // once), and no other warp reads row 0's record (only a finalizer reads records, and
        // it is this warp), so no record, no release and no returned value: the state and the
        // claim hint are updated fire-and-forget for the scheduler's scans and dead checks.
        if (lane == 0) {
            atomicMin(a.roll_first + b, 0);
            red_or_relaxed(a.roll_state + b, 1ull | (1ull << 32));
        }
        F = 0;
    } else {
        if (lane == 0) {
            const int64_t r = base + j;
            // A finalizer reads the record of the deciding row F (status, candidate) and, only
            // when the caller asked for them, the normalisers / Z of rows 0..F.  An accepted row
            // (never F) without those outputs therefore stores nothing and needs no release.
            const bool outs = a.out_norm != nullptr || a.out_z != nullptr;
            if (decides) {
                a.row_status[r] = status;
                a.row_cand[r] = cand;
            }
            if (outs) {
                a.row_z[r] = z;
                a.row_norm[r] = norm;
            }
            if (decides) atomicMin(a.roll_first + b, j);  // claim hint only (relaxed)
            const unsigned long long mine = (1ull << j) | (decides ? (1ull << (32 + j)) : 0ull);
            // release: this row's record; acquire: every earlier row's record of the rollout
            const unsigned long long old = (decides || outs) ? atom_or_acq_rel(a.roll_state + b, mine)
                                                             : atom_or_acquire(a.roll_state + b, mine);
            int F0, F1;
            if (!prefix_decided(old, F0) && prefix_decided(old | mine, F1)) F = F1;
        }
        F = __shfl_sync(0xFFFFFFFFu, F, 0);
    }
    if (F < 0) return false;
    __syncwarp();  // lane 0's acquire orders the other lanes' reads below
    const int32_t* d = a.draft + (int64_t)b * a.k;
    int32_t dl = -1, stF = status, cF = cand;
    float nl = 0.f;
    unsigned long long zl = 0ull;
    // d_{F+1} is needed only for an accepted EOS at row F (this row's status is known)
    if (lane < F || (lane == F && lane < q && (F != j || status == ST_EOS))) dl = (dpf != DPF_NONE) ? dpf : d[lane];
    if (lane <= F && (a.out_norm || a.out_z)) {
        nl = (lane == j) ? norm : __ldcg(a.row_norm + base + lane);
        zl = (lane == j) ? z : __ldcg(a.row_z + base + lane);
    }
    if (lane == F && F != j) {
        stF = __ldcg(a.row_status + base + F);
        cF = __ldcg(a.row_cand + base + F);
    }
    stF = __shfl_sync(0xFFFFFFFFu, stF, F);
    if (stF == ST_ERR) {  // a needed row is invalid (R0): the step emits nothing (the commit stops it)
        cF = __shfl_sync(0xFFFFFFFFu, cF, F);
        if (lane < kp1) a.out_tokens[base + lane] = -1;
        tok = -1;
        no = 0;
        if (lane == 0) {
            atomicOr(a.dev_err, (uint32_t)cF);
            a.out_len[b] = 0;
            a.out_acc[b] = 0;
            if (a.sctl) atomicAdd(a.sctl + SC_DONE, 1u);
        }
        return true;
    }
    // Alg. 1 lines 10-31: d_1..d_F accepted, then the sample of row F (or its accepted EOS)
    tok = (lane < F) ? dl : ((lane == F) ? (stF == ST_EOS ? dl : cF) : -1);
    no = F + 1;
    const int acc = (stF == ST_EOS) ? F + 1 : F;
    if (lane < kp1) a.out_tokens[base + lane] = tok;
    if (lane <= F) {
        if (a.out_norm) a.out_norm[base + lane] = nl;
        if (a.out_z) a.out_z[base + lane] = zl;
    }
    if (lane == 0) {
        a.out_len[b] = no;
        a.out_acc[b] = acc;
        if (q > 0) {
            stat[STAT_STEPS_SPEC] += 1ull;
            stat[STAT_EMIT_SPEC] += (unsigned long long)no;
            stat[STAT_ACCEPTED] += (unsigned long long)acc;
            stat[STAT_PROPOSED] += (unsigned long long)q;
            stat[STAT_HIST + min(no, STAT_HIST_BINS - 1)] += 1ull;
        } else {
            stat[STAT_STEPS_PLAIN] += 1ull;
            stat[STAT_EMIT_PLAIN] += (unsigned long long)no;
        }
        stat[STAT_ROWS_NEEDED] += (unsigned long long)(F + 1);
        if (a.sctl) {
            const unsigned dn = atomicAdd(a.sctl + SC_DONE, 1u);  // scheduler termination count
            TRACE(TR_FIN, (int)dn, b, F);
        }
    }
    return true;
}

// Claim the next needed row of the plan's j-major table (Alg. 1's order across the batch),
// skipping rows at or above an already-decided row of their rollout.  b < 0: none left.
__device__ RowDesc claim_row(const VerifyArgs& a, int rows, int base = 0) {
    for (;;) {
        const int r = base + (int)atomicAdd(a.ctl + VCTL_NEXT, 1u);
        if (r >= rows) break;
        const RowDesc it = a.items[r];
        if (it.j > ld_volatile_i32(a.roll_first + it.b)) continue;  // decided below
        return it;
    }
    RowDesc none;
    none.b = -1;
    return none;
}

// ================================================================ epilogue warp
// Decision, sample and bookkeeping of one row (one warp).
__device__ void epilogue_row(const VerifyArgs& a, VShared& sh, const EpiBuf& E, int lane) {
    const RowDesc& dsc = E.dsc;
    const int b = dsc.b, j = dsc.j, q = dsc.q, d = dsc.d;
    const bool ok = E.ok != 0;
    const uint16_t* row = a.logits + dsc.rowno * a.stride;
    const int nb = a.ngroup * NCW;  // blocks in element order: i = g*NCW + w
    int status = ST_DECIDED, cand = -1;
    unsigned long long Zo = 0;
    float norm = 0.f;
    if (a.T == 0.f) {  // greedy (R1)
        int g = (lane < NCW) ? (int)(uint32_t)E.csum[0][lane] : 0x7FFFFFFF;
#pragma unroll
        for (int mm = 16; mm; mm >>= 1) g = min(g, __shfl_xor_sync(0xFFFFFFFFu, g, mm));
        g = ok ? g : -1;
        const bool acc = ok && j < q && d == g;
        status = acc ? ((a.eos >= 0 && d == a.eos) ? ST_EOS : ST_CONT) : ST_DECIDED;
        cand = g;
        Zo = ok ? 1ull : 0ull;
        norm = ok ? 1.f : 0.f;
    } else if (ok) {
        MassParams mp;
        mp.c = a.c;
        mp.nmc = -__fmul_rn(E.m, a.c);
        mp.clampv = -(float)(a.S + 2);
        mp.magic = 12582912.0f + (float)a.S;
        // lane l owns the contiguous block range [l*per, (l+1)*per)
        const int per = (nb + 31) / 32;
        const int i0 = min(nb, lane * per), i1 = min(nb, i0 + per);
        uint64_t ls = 0;
        for (int i = i0; i < i1; ++i) ls += E.csum[i / NCW][i % NCW];
        const uint64_t incl = warp_incl_scan_u64(ls, lane);
        const uint64_t Z = shfl_u64(incl, 31);
        const uint64_t md = (d >= 0) ? mass_of(__uint_as_float((uint32_t)row[d] << 16), mp) : 0ull;
        bool acc = false;
        if (j < q) acc = uniform_floor(row_draw(a, dsc, PURPOSE_ACCEPT), Z) < md;
        status = acc ? ((a.eos >= 0 && d == a.eos) ? ST_EOS : ST_CONT) : ST_DECIDED;
        Zo = Z;
        norm = (float)ldexp((double)Z, -a.S);
        if (status == ST_DECIDED) {
            // residual (d excluded) or bonus sample (R8) by inverse CDF in ascending id
            const int excl = (j < q) ? d : -1;
            const uint64_t U = uniform_floor(row_draw(a, dsc, PURPOSE_SAMPLE), Z - ((j < q) ? md : 0ull));
            // the excluded token's mass comes off the block holding it
            const int ex_blk = (excl >= 0) ? ((excl / (2 * CHE)) * NCW + ((excl % (2 * CHE)) / CHE) * (NCW / 2) +
                                              ((excl % CHE) / BLK))
                                           : -1;
            const uint64_t ex_lane_adj = (ex_blk >= i0 && ex_blk < i1) ? md : 0ull;
            const uint64_t incl2 = warp_incl_scan_u64(ls - ex_lane_adj, lane);
            const unsigned hit = __ballot_sync(0xFFFFFFFFu, U < incl2);
            const int L = hit ? (__ffs(hit) - 1) : 31;
            int xb = 0;
            uint64_t ub = 0;
            if (lane == L) {  // the crossing block inside lane L's range
                uint64_t cum = incl2 - (ls - ex_lane_adj);
                for (int i = i0; i < i1; ++i) {
                    const uint64_t bsum = E.csum[i / NCW][i % NCW] - ((i == ex_blk) ? md : 0ull);
                    if (U < cum + bsum) {
                        xb = i;
                        ub = U - cum;
                        break;
                    }
                    cum += bsum;
                }
            }
            xb = __shfl_sync(0xFFFFFFFFu, xb, L);
            ub = shfl_u64(ub, L);
            const int g = xb / NCW, w = xb % NCW;
            const int e_blk = 2 * g * CHE + (w / (NCW / 2)) * CHE + (w % (NCW / 2)) * BLK;
            // rescan the block from L2: lane l owns 32 contiguous elements
            const int e0 = lane * EPL;
            auto load8 = [&](int t) {
                const int e = e_blk + e0 + t * 8;
                uint4 v = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
                if (dsc.aligned && e + 8 <= a.V) {
                    v = __ldg(reinterpret_cast<const uint4*>(row + e));
                } else {
                    uint16_t t8[8];
                    for (int i = 0; i < 8; ++i) t8[i] = (e + i < a.V) ? row[e + i] : (uint16_t)0xFF80u;
                    v.x = t8[0] | ((uint32_t)t8[1] << 16);
                    v.y = t8[2] | ((uint32_t)t8[3] << 16);
                    v.z = t8[4] | ((uint32_t)t8[5] << 16);
                    v.w = t8[6] | ((uint32_t)t8[7] << 16);
                }
                return v;
            };
            uint64_t lsum = 0;
            for (int t = 0; t < EPL / 8; ++t) {
                const uint4 v8 = load8(t);
                uint64_t mm[8];
                mass8_masked(v8, mp, e0 + t * 8, a.V - e_blk, excl - e_blk, mm);
#pragma unroll
                for (int i = 0; i < 8; ++i) lsum += mm[i];
            }
            const uint64_t inc3 = warp_incl_scan_u64(lsum, lane);
            const unsigned hit3 = __ballot_sync(0xFFFFFFFFu, ub < inc3);
            const int L3 = hit3 ? (__ffs(hit3) - 1) : 31;
            int tok = -1;
            if (lane == L3) {  // reload and recompute this lane's masses in order
                uint64_t cum = inc3 - lsum;
                for (int t = 0; t < EPL / 8 && tok < 0; ++t) {
                    uint64_t mm[8];
                    mass8_masked(load8(t), mp, e0 + t * 8, a.V - e_blk, excl - e_blk, mm);
                    for (int i = 0; i < 8; ++i) {
                        cum += mm[i];
                        if (tok < 0 && cum > ub) tok = e_blk + e0 + t * 8 + i;
                    }
                }
            }
            cand = __shfl_sync(0xFFFFFFFFu, tok, L3);
        }
    }
    if (lane == 0) {
        sh.stat[STAT_ROWS_VERIFIED] += 1ull;
        complete_row(a, sh.stat, b, j, q, ok ? status : ST_ERR, ok ? cand : (int)E.err, Zo, norm);
    }
    __syncwarp();
}

__global__ void __launch_bounds__(NTHR, CTAS_PER_SM) verify_rows_kernel(const VerifyArgs a) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint16_t* ring = reinterpret_cast<uint16_t*>(smem_raw);
    VShared& sh = *reinterpret_cast<VShared*>(smem_raw + (size_t)NSTAGE * CHE * 2);
    pdl_wait();  // dependents launch at exit (the cluster kernel plans before its wait)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rows = (int)a.ctl[VCTL_ROWS];

    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&sh.full[i], 1);
            mbar_init(&sh.empty[i], NCW / 2);  // the 8 warps of the stage's half
        }
        for (int i = 0; i < RF; ++i) {
            mbar_init(&sh.rfull[i], 1);
            mbar_init(&sh.rempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sh.efull[i], NCW);  // every consumer warp hands its block sums over
            mbar_init(&sh.eempty[i], 1);
        }
        fence_mbar_init();
    }
    for (int i = tid; i < STAT_COUNT; i += NTHR) sh.stat[i] = 0ull;
    __syncthreads();

    if (warp == PROD_WARP) {
        // ======================================================== producer warp
        if (lane != 0) return;
        const uint64_t pol_keep = 0;  // pass 1: default L2 policy (the row is re-read)
        const uint64_t pol_first = policy_evict_first();
        uint32_t rph = 0;    // row-empty phase bits, one per FIFO slot
        uint32_t P = 0;      // chunks issued so far: stage P % NSTAGE, use P / NSTAGE
        auto claim = [&]() { return claim_row(a, rows); };
        RowDesc nxt = claim();
        for (int seq = 0;; ++seq) {
            const RowDesc cur = nxt;
            const int f = seq % RF;
            if (seq >= RF) {
                mbar_wait(&sh.rempty[f], (rph >> f) & 1u);
                rph ^= 1u << f;
            }
            sh.desc[f] = cur;
            mbar_arrive(&sh.rfull[f]);  // release: the descriptor is visible to the consumers
            if (cur.b < 0) break;
            const uint16_t* row = a.logits + cur.rowno * a.stride;
            const bool aligned = cur.aligned != 0;
            for (int pass = 0; pass < 2; ++pass) {
                // (claiming the following row earlier, under pass 1, raises speculative
                // row reads more than it hides claim latency: measured slower)
                if (pass == 1 && c_claim_early) nxt = claim();
                for (int c = 0; c < 2 * a.ngroup; ++c, ++P) {
                    const int s = (int)(P % NSTAGE);
                    // a stage's k-th fill waits for its (k-1)-th release (first fill: free)
                    mbar_wait(&sh.empty[s], ((P / NSTAGE) & 1u) ^ 1u);
                    const int cv = max(0, min(CHE, a.V - c * CHE));  // valid elements
                    const int bulk = aligned ? (cv & ~7) : 0;
                    uint16_t* dst = ring + (size_t)s * CHE;
                    fence_proxy_async_smem();
                    if (bulk) {
                        mbar_arrive_expect_tx(&sh.full[s], (uint32_t)bulk * 2u);
                        bulk_g2s(dst, row + (size_t)c * CHE, (uint32_t)bulk * 2u, &sh.full[s],
                                 pass ? pol_first : pol_keep);
                    } else {
                        mbar_arrive(&sh.full[s]);
                    }
                }
            }
            if (!c_claim_early) nxt = claim();
        }
        return;
    }

    if (warp == EPI_WARP) {
        // ======================================================== epilogue warp
        for (int seq = 0;; ++seq) {
            const int e = seq & 1;
            mbar_wait(&sh.efull[e], (seq >> 1) & 1);
            if (sh.epi[e].dsc.b < 0) break;
            epilogue_row(a, sh, sh.epi[e], lane);
            if (lane == 0) mbar_arrive(&sh.eempty[e]);
        }
        __syncwarp();
        if (a.stats && lane == 0)
            for (int i = 0; i < STAT_COUNT; ++i)
                if (sh.stat[i]) atomicAdd(a.stats + i, sh.stat[i]);
        return;
    }

    // ============================================================ consumer warps
    const int half = warp / (NCW / 2);         // warps 0-7: even chunk, 8-15: odd chunk
    const int wblk = (warp % (NCW / 2)) * BLK; // this warp's 1024-element block in the chunk
    MassParams mp;
    mp.c = a.c;
    mp.clampv = -(float)(a.S + 2);
    mp.magic = 12582912.0f + (float)a.S;
    uint32_t u = 0;  // chunks consumed so far (CTA-uniform): stage u % NSTAGE, use u / NSTAGE
#ifdef BS_PHASE_TIMING
    long long ph_t = clock64();
#endif
    for (int seq = 0;; ++seq) {
        const int f = seq % RF;
        const int e = seq & 1;
        mbar_wait(&sh.rfull[f], (seq / RF) & 1);
        const RowDesc dsc = sh.desc[f];
        // the epilogue must be done with the record this row will fill (row seq - 2)
        mbar_wait(&sh.eempty[e], ((seq >> 1) & 1) ^ 1);
        EpiBuf& E = sh.epi[e];
        if (dsc.b < 0) {  // end: pass the marker on to the epilogue warp
            if (tid == 0) E.dsc.b = -1;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh.efull[e]);
            break;
        }
        const uint16_t* row = a.logits + dsc.rowno * a.stride;
        PH_MARK(0);

        // ---------------------------------------------------- pass 1: row max
        uint32_t mx = 0xFF80FF80u;
        for (int g = 0; g < a.ngroup; ++g) {
            const int c = 2 * g + half;
            const uint32_t uc = u + (uint32_t)c;
            const int sg = (int)(uc % NSTAGE);
            mbar_wait(&sh.full[sg], (uc / NSTAGE) & 1u);
            const uint16_t* buf = ring + (size_t)sg * CHE;
            const int cv = max(0, min(CHE, a.V - c * CHE));
            const int bulk = dsc.aligned ? (cv & ~7) : 0;
            if (cv == CHE && bulk == CHE) {
#pragma unroll
                for (int t = 0; t < TPW; ++t) {
                    const uint4 v = lds128(buf + wblk + t * 256 + lane * 8);
                    mx = hmax2_nan_u32(mx, v.x);
                    mx = hmax2_nan_u32(mx, v.y);
                    mx = hmax2_nan_u32(mx, v.z);
                    mx = hmax2_nan_u32(mx, v.w);
                }
            } else {  // partial / unaligned chunk: element-wise from smem or global
                for (int t = 0; t < TPW; ++t) {
                    const int e0 = wblk + t * 256 + lane * 8;
                    for (int i = 0; i < 8; ++i) {
                        const int el = e0 + i;
                        if (el < cv) {
                            const uint16_t v = (el < bulk) ? buf[el] : row[(size_t)c * CHE + el];
                            mx = hmax2_nan_u32(mx, (uint32_t)v | 0xFF800000u);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh.empty[sg]);
        }
        u += 2u * (uint32_t)a.ngroup;
        {
            const float lo = bf16lo(mx), hi = bf16hi(mx);
            uint32_t bad = (isnan(lo) || isnan(hi) || lo == INFINITY || hi == INFINITY) ? 1u : 0u;
            float fm = fmaxf(lo, hi);
#pragma unroll
            for (int mm = 16; mm; mm >>= 1) fm = fmaxf(fm, __shfl_xor_sync(0xFFFFFFFFu, fm, mm));
            bad = __any_sync(0xFFFFFFFFu, bad) ? 1u : 0u;
            if (lane == 0) {
                sh.wmax[warp] = fm;
                sh.wbad[warp] = bad;
            }
        }
        named_bar(1, NCT);
        PH_MARK(1);
        float m = -INFINITY;
        uint32_t bb = 0;
        for (int w = 0; w < NCW; ++w) {
            m = fmaxf(m, sh.wmax[w]);
            bb |= sh.wbad[w];
        }
        bool ok = true;
        uint32_t err = 0;
        if (bb) { ok = false; err |= DEV_BAD_LOGIT; }
        else if (m == -INFINITY) { ok = false; err |= DEV_ALL_NEGINF; }
        else if (a.T > 0.f && !(fabsf(__fmul_rn(m, a.c)) < 16777216.0f)) { ok = false; err |= DEV_RANGE; }
        if (tid == 0) {
            mbar_arrive(&sh.rempty[f]);  // (error bits reported at finalize if the row is needed)  // the descriptor slot is free (register copy kept)
            E.dsc = dsc;
            E.m = m;
            E.ok = ok ? 1 : 0;
            E.err = err;
        }
        mp.nmc = -__fmul_rn(m, a.c);

        // ---------------------------------------------------- pass 2: masses / argmax
        int first = 0x7FFFFFFF;
        for (int g = 0; g < a.ngroup; ++g) {
            const int c = 2 * g + half;
            const uint32_t uc = u + (uint32_t)c;
            const int sg = (int)(uc % NSTAGE);
            mbar_wait(&sh.full[sg], (uc / NSTAGE) & 1u);
            const uint16_t* buf = ring + (size_t)sg * CHE;
            const int cv = max(0, min(CHE, a.V - c * CHE));
            const int bulk = dsc.aligned ? (cv & ~7) : 0;
            if (a.T == 0.f) {  // greedy (R1): the first index attaining the max
                if (ok && first == 0x7FFFFFFF) {
                    for (int t = 0; t < TPW; ++t) {
                        const int e0 = wblk + t * 256 + lane * 8;
                        int fi = 0x7FFFFFFF;
                        for (int i = 7; i >= 0; --i) {
                            const int el = e0 + i;
                            if (el < cv) {
                                const uint16_t v = (el < bulk) ? buf[el] : row[(size_t)c * CHE + el];
                                if (__uint_as_float((uint32_t)v << 16) == m) fi = c * CHE + el;
                            }
                        }
#pragma unroll
                        for (int mm = 16; mm; mm >>= 1) fi = min(fi, __shfl_xor_sync(0xFFFFFFFFu, fi, mm));
                        if (fi != 0x7FFFFFFF) {
                            first = fi;
                            break;
                        }
                    }
                }
            } else {
                uint64_t acc = 0;
                if (ok) {
                    if (cv == CHE && bulk == CHE) {
#pragma unroll
                        for (int t = 0; t < TPW; t += 4) {  // 4 tiles = 16 independent pair chains
                            const uint4 v0 = lds128(buf + wblk + t * 256 + lane * 8);
                            const uint4 v1 = lds128(buf + wblk + (t + 1) * 256 + lane * 8);
                            const uint4 v2 = lds128(buf + wblk + (t + 2) * 256 + lane * 8);
                            const uint4 v3 = lds128(buf + wblk + (t + 3) * 256 + lane * 8);
                            acc += (mass8(v0, mp) + mass8(v1, mp)) + (mass8(v2, mp) + mass8(v3, mp));
                        }
                    } else {
                        for (int t = 0; t < TPW; ++t) {
                            const int e0 = wblk + t * 256 + lane * 8;
                            for (int i = 0; i < 8; ++i) {
                                const int el = e0 + i;
                                if (el < cv) {
                                    const uint16_t v = (el < bulk) ? buf[el] : row[(size_t)c * CHE + el];
                                    acc += mass_of(__uint_as_float((uint32_t)v << 16), mp);
                                }
                            }
                        }
                    }
                }
                const uint64_t bs = warp_sum_u51(acc);
                if (lane == 0) E.csum[g][warp] = bs;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sh.empty[sg]);
        }
        u += 2u * (uint32_t)a.ngroup;
        if (a.T == 0.f && lane == 0) E.csum[0][warp] = (unsigned long long)(uint32_t)first;
        __syncwarp();
        if (lane == 0) mbar_arrive(&sh.efull[e]);  // release: block sums -> epilogue
        PH_MARK(2);
#ifdef BS_PHASE_TIMING
        if (tid == 0) atomicAdd(&g_phase[15], 1ull);
#endif
    }
}

#include "verify_cluster.cuh"
#include "verify_topp.cuh"

// ---- plan: clamp q per rollout, reset per-rollout state, and lay out the step's rows as a
// j-major table (rows (b, 0) of every live rollout, then (b, 1), ...: Alg. 1's order across
// the batch) with everything a row needs (no dependent loads when a CTA claims it).
constexpr int PLAN_NT = 1024;
__global__ void __launch_bounds__(PLAN_NT) verify_plan_kernel(
    int n, int k, int V, const int32_t* slots, const int32_t* draft, const int32_t* draft_len,
    const int32_t* pos, const int32_t* max_len, const int32_t* finished,
    const unsigned long long* uid, const uint16_t* logits, const int64_t* row_index,
    int64_t stride, int32_t* rb_q, RowDesc* items, unsigned int* ctl, int32_t* roll_first,
    unsigned long long* roll_state, int32_t* out_len, int32_t* out_acc, int32_t* out_tokens,
    float* out_norm, unsigned long long* out_z, uint32_t* dev_err, int mode) {
    __shared__ int hist[33], lvl_off[33], lvl_ctr[33], s_rows, s_nact;
    pdl_wait();  // dependents launch at exit (the cluster kernel plans before its wait)
    const int tid = threadIdx.x;
    if (tid < 33) {
        hist[tid] = 0;
        lvl_ctr[tid] = 0;
    }
    __syncthreads();
    const int per = (n + PLAN_NT - 1) / PLAN_NT;
    const int b0 = min(n, tid * per), b1 = min(n, b0 + per);
    const int kp1 = k + 1;
    for (int b = b0; b < b1; ++b) {
        const int s = slots[b];
        const int p = pos[s], L = max_len[s];
        int q = -1;
        if (!finished[s] && p < L) {
            q = min(max(draft_len[b], 0), min(k, L - p - 1));
            for (int i = 0; i < q; ++i) {
                const int t = draft[(int64_t)b * k + i];
                if (t < 0 || t >= V) {
                    atomicOr(dev_err, DEV_BAD_DRAFT);
                    q = -1;
                    break;
                }
            }
        }
        rb_q[b] = q;
        roll_first[b] = q;  // the bonus row q always decides; earlier rows may lower it
        roll_state[b] = 0ull;
        if (q >= 0) atomicAdd(&hist[q], 1);
        for (int jj = 0; jj < kp1; ++jj) {
            if (out_norm) out_norm[(int64_t)b * kp1 + jj] = 0.f;
            if (out_z) out_z[(int64_t)b * kp1 + jj] = 0ull;
        }
        if (q < 0) {
            out_len[b] = 0;
            out_acc[b] = 0;
            for (int jj = 0; jj < kp1; ++jj) out_tokens[(int64_t)b * kp1 + jj] = -1;
        }
    }
    __syncthreads();
    if (tid == 0) {  // level j holds the rollouts with q >= j
        int off = 0, nact = 0;
        for (int j = 0; j <= k; ++j) {
            int cnt = 0;
            for (int qq = j; qq <= k; ++qq) cnt += hist[qq];
            if (j == 0) nact = cnt;
            lvl_off[j] = off;
            off += cnt;
        }
        s_rows = off;
        s_nact = nact;
    }
    __syncthreads();
    for (int b = b0; b < b1; ++b) {
        const int q = rb_q[b];
        if (q < 0) continue;
        const int s = slots[b];
        const unsigned long long u = uid[s];
        const int p = pos[s];
        for (int j = 0; j <= q; ++j) {
            RowDesc it;
            it.b = b;
            it.j = j;
            it.q = q;
            it.d = (j < q) ? draft[(int64_t)b * k + j] : -1;
            it.rowno = row_index ? row_index[(int64_t)b * kp1 + j] : (int64_t)b * kp1 + j;
            it.uid = u;
            it.position = p + j;
            it.aligned = ((reinterpret_cast<uintptr_t>(logits + it.rowno * stride) & 15u) == 0) ? 1 : 0;
            it.pad[0] = it.pad[1] = 0;
            items[lvl_off[j] + atomicAdd(&lvl_ctr[j], 1)] = it;  // order within a level: any
        }
    }
    if (tid == 0) {
        ctl[VCTL_NEXT] = 0u;
        ctl[VCTL_NACTIVE] = (unsigned)s_nact;
        ctl[VCTL_ROWS] = (unsigned)s_rows;
        ctl[VCTL_MODE] = (unsigned)mode;
    }
}

// Which kernel verifies rows (bsx_set_verify_kernel; env BS_VERIFY_KERNEL for tools).
enum { VK_AUTO = 0, VK_ROWS = 1, VK_CLUSTER = 3 };  // (2: the unpipelined split kernel, removed)
static int verify_kind(const bs_ctx* ctx, int V) {
    int k = ctx->verify_kind;
    if (k == VK_AUTO) k = ctx->env_kind;
    if (k == VK_AUTO) k = VK_CLUSTER;
    if (k == VK_CLUSTER && (V + CK_CL - 1) / CK_CL > CK_MAXSL) k = VK_ROWS;
    return k;
}
// Slice of a row per cluster CTA: ceil(V / 8) rounded up to whole 512-element tiles.
static int cluster_slice(int V) { return ((V + CK_CL - 1) / CK_CL + CK_TILE - 1) / CK_TILE * CK_TILE; }

// Slice of a filtered row per cluster CTA: ceil(V / 8) rounded up to whole 256-element tiles.
static int topp_slice(int V) { return ((V + TP_CL - 1) / TP_CL + 255) / 256 * 256; }
static int ntile_ok(int V) { return topp_slice(V) / 256 <= TP_MAXLT ? 1 : 0; }

cudaError_t launch_verify(bs_ctx* ctx, int32_t n, const int32_t* slots, const void* logits,
                          const int64_t* row_index, int64_t stride, const int32_t* draft,
                          const int32_t* draft_len, int32_t k, float T, float top_p, int32_t top_k,
                          int32_t* out_tokens, int32_t* out_len, int32_t* out_acc,
                          float* out_norm, unsigned long long* out_z, cudaStream_t st,
                          int32_t* commit_finished, bool* committed, const LookupArgs* lookup,
                          bool* looked_up) {
    if (committed) *committed = false;
    if (looked_up) *looked_up = false;
    if (n == 0) return cudaSuccess;
    const int V = ctx->cfg.vocab;
    if (top_k >= V) top_k = 0;  // keeps every token
    const bool topp = T > 0.f && (top_p < 1.f || top_k > 0);  // filtered rows (R5k, R5)
    const int kind = topp ? VK_ROWS : verify_kind(ctx, V);
    cudaError_t e = cudaSuccess;
    // the cluster kernel plans in-kernel (each rollout's row-0 claimer); the others take the
    // plan kernel's j-major row table
    if (kind != VK_CLUSTER) e = launch_pdl(
        verify_plan_kernel, dim3(1), dim3(PLAN_NT), 0, st, n, k, V, slots, draft, draft_len,
        (const int32_t*)ctx->pos.p, (const int32_t*)ctx->max_len.p,
        (const int32_t*)ctx->finished.p, (const unsigned long long*)ctx->uid.p,
        static_cast<const uint16_t*>(logits), row_index, stride, ctx->rb_q.p,
        reinterpret_cast<RowDesc*>(ctx->vqueue.p), ctx->vctl.p, ctx->vroll_first.p,
        ctx->vroll_state.p, out_len, out_acc, out_tokens, out_norm, out_z, ctx->dev_err.p, 0);
    if (e != cudaSuccess) return e;
    VerifyArgs a = {};
    a.slots = slots;
    a.logits = static_cast<const uint16_t*>(logits);
    a.row_index = row_index;
    a.stride = stride;
    a.draft = draft;
    a.k = k;
    a.V = V;
    a.S = ctx->S;
    a.eos = ctx->cfg.eos_id;
    a.nchunk = (V + CHE - 1) / CHE;
    a.ngroup = (a.nchunk + 1) / 2;
    if (a.ngroup > MAXG) return cudaErrorInvalidValue;
    a.T = T;
    a.c = (T > 0.f) ? (float)(1.4426950408889634 / (double)T) : 0.f;
    a.seed = ctx->cfg.seed;
    a.pos = ctx->pos.p;
    a.uid = ctx->uid.p;
    a.rb_q = ctx->rb_q.p;
    a.items = reinterpret_cast<const RowDesc*>(ctx->vqueue.p);
    a.ctl = ctx->vctl.p;
    a.dev_err = ctx->dev_err.p;
    a.row_status = ctx->vrow_status.p;
    a.row_cand = ctx->vrow_cand.p;
    a.row_z = ctx->vrow_z.p;
    a.row_norm = ctx->vrow_norm.p;
    a.roll_first = ctx->vroll_first.p;
    a.roll_state = ctx->vroll_state.p;
    a.out_tokens = out_tokens;
    a.out_len = out_len;
    a.out_acc = out_acc;
    a.out_norm = out_norm;
    a.out_z = out_z;
    a.stats = ctx->stats.p;
    if (kind == VK_CLUSTER && !topp) {
        a.n = n;
        a.draft_len = draft_len;
        a.max_len = ctx->max_len.p;
        a.finished = ctx->finished.p;
        a.sctl = ctx->vctl.p;
        a.next_row = ctx->vnext_row.p;
        a.rrec = ctx->vrrec.p;
        a.live = ctx->vlive.p;
        a.eager_ok = ctx->env_eager;
        a.early_plan = ctx->early_plan;
        a.rs_key = ctx->rs_key;
        a.rs_bad = ctx->rs_bad;
        if (committed) {  // fused commit (bs_verify_commit)
            a.commit = 1;
            a.M = ctx->M;
            a.c_tail = ctx->tail.p;
            a.c_ctx_len = ctx->ctx_len.p;
            a.c_pos = ctx->pos.p;
            a.c_finished = ctx->finished.p;
            a.c_fin_out = commit_finished;
            a.c_resp = ctx->responses;
            a.c_resp_stride = ctx->resp_stride;
            *committed = true;
            if (lookup && looked_up) {  // fused lookup (bs_verify_commit_lookup)
                a.lookup = 1;
                a.lk = *lookup;
                *looked_up = true;
            }
        }
    }
    if (topp) {  // R5k / R5: top-k / top-p filtered rows (verify_topp.cuh)
        if (ntile_ok(V) == 0) return cudaErrorInvalidValue;
        // the slice staged in shared memory when it fits beside TopPShared at two CTAs per SM
        const size_t staged_sm = tp_shared_bytes() + (size_t)topp_slice(V) * 2;
        const int staged = staged_sm <= TP_STAGE_MAX ? 1 : 0;
        const size_t tsm = staged ? staged_sm : tp_shared_bytes();
        if (ctx->kcfg_topp != (int)tsm) {
            e = cudaFuncSetAttribute(verify_topp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)tsm);
            if (e != cudaSuccess) return e;
            ctx->kcfg_topp = (int)tsm;
        }
        // one 8-CTA cluster per row in flight (two CTAs per SM)
        const int tcl = std::max(1, std::min((ctx->num_sms * 2) / TP_CL, n * (k + 1)));
        return launch_pdl(verify_topp_kernel, dim3(tcl * TP_CL), dim3(TP_NT), tsm, st, a, top_p, top_k,
                          topp_slice(V), staged);
    }
    if (kind == VK_CLUSTER) {
        const int SL = cluster_slice(V);
        const size_t csm = ck_smem_bytes(SL);
        if (ctx->kcfg_cluster_smem != csm) {
            e = cudaFuncSetAttribute(verify_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)csm);
            if (e != cudaSuccess) return e;
            if (CK_CL > 8) {
                e = cudaFuncSetAttribute(verify_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                if (e != cudaSuccess) return e;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(CK_CL * ctx->num_sms);
            cfg.blockDim = dim3(CK_NT);
            cfg.dynamicSmemBytes = csm;
            int ncl = 0;
            e = cudaOccupancyMaxActiveClusters(&ncl, verify_cluster_kernel, &cfg);
            if (e != cudaSuccess) return e;
            ctx->kcfg_clusters = std::max(1, ncl);
            ctx->kcfg_cluster_smem = csm;
        }
        const int ncl_use = ctx->max_clusters > 0 ? std::min(ctx->max_clusters, ctx->kcfg_clusters)
                                                  : ctx->kcfg_clusters;
        a.ncl = ncl_use;
        const dim3 grid(ncl_use * CK_CL);
        if (ctx->kcfg_coop < 0) {  // probe once, outside stream capture (a failed launch would end it)
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            cudaStreamIsCapturing(st, &cs);
            if (cs == cudaStreamCaptureStatusNone) {
                e = launch_pdl_ex(true, verify_cluster_kernel, grid, dim3(CK_NT), csm, st, a, SL);
                if (e == cudaSuccess) {
                    ctx->kcfg_coop = 1;
                    return e;
                }
                cudaGetLastError();
                ctx->kcfg_coop = 0;
            }
        }
        return launch_pdl_ex(ctx->kcfg_coop == 1, verify_cluster_kernel, grid, dim3(CK_NT), csm, st, a, SL);
    }
    const size_t smem = (size_t)NSTAGE * CHE * 2 + sizeof(VShared);
    if (!ctx->kcfg_rows) {
        e = cudaFuncSetAttribute(verify_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        ctx->kcfg_rows = 1;
    }
    const int grid = std::max(1, std::min(ctx->num_sms * CTAS_PER_SM, n * (k + 1)));
    return launch_pdl(verify_rows_kernel, dim3(grid), dim3(NTHR), smem, st, a);
}

}  // namespace bs

// Event trace of the cluster kernel (BS_TRACE builds): copies up to max_ev uint4 events to
// host memory out, returns the number recorded (and resets the trace when reset != 0).
extern "C" int bsx_trace_read(void* out, int max_ev, int reset) {
#ifdef BS_TRACE
    // compacts the nonzero events (per-CTA slices) into out
    static uint4* host = nullptr;
    if (!host) host = (uint4*)malloc(sizeof(uint4) << 20);
    cudaMemcpyFromSymbol(host, bs::g_trace, sizeof(uint4) << 20);
    int m = 0;
    for (int i = 0; i < (1 << 20) && m < max_ev; ++i)
        if (host[i].z | host[i].w) static_cast<uint4*>(out)[m++] = host[i];
    if (reset) {
        memset(host, 0, sizeof(uint4) << 20);
        cudaMemcpyToSymbol(bs::g_trace, host, sizeof(uint4) << 20);
    }
    return m;
#else
    (void)out;
    (void)max_ev;
    (void)reset;
    return -1;
#endif
}

extern "C" int bsx_phase_times(unsigned long long* out16, int reset) {
#ifdef BS_PHASE_TIMING
    cudaMemcpyFromSymbol(out16, bs::g_phase, sizeof(unsigned long long) * 16);
    if (reset) {
        unsigned long long z[16] = {0};
        cudaMemcpyToSymbol(bs::g_phase, z, sizeof z);
    }
    return 1;
#else
    (void)out16;
    (void)reset;
    return 0;
#endif
}
