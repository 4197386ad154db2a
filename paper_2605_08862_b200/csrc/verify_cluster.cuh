// verify_cluster.cuh — the verify + resample kernel (reading R, Eq. 2-3, Alg. 1) for every
// batch size: each logits row is split across an 8-CTA thread-block cluster and streamed
// through shared memory once.  Included by verify.cu inside namespace bs.
//
// Per CTA (320 threads): slice [rank*SL, rank*SL + SL) of every row the cluster verifies.
//   * PRODUCER warp (lane 0).  In the leader CTA it also claims rows from the plan's j-major
//     table just in time (when its slice buffer frees) and broadcasts each descriptor to the
//     8 CTAs with st.async (mbarrier completion).  Every producer bulk-copies (TMA) its slice
//     of the row into one of two shared-memory buffers.
//   * 2 MAX warps run one row ahead: pass 1 (slice max; greedy: its lowest index) of row
//     i+1, published to the 8 CTAs (16-byte st.async into a 4-deep ring), while
//   * 6 MASS warps do pass 2 of row i: integer masses from shared memory with the cluster
//     max, 512-element tile sums kept locally, the slice sum and mass(d) published the same
//     way; then the buffer is freed.  The row is read from HBM exactly once.
//   * EPILOGUE warp.  Z, mass(d), the accept test (Philox (pos+j, ACCEPT)), the
//     residual/bonus sample (the crossing slice from the 8 slice sums, the crossing tile from
//     the local tile sums, one tile re-read from L2), then the rollout's completion protocol.
// Ring reuse is safe without extra handshakes: a CTA cannot publish row i+4 before every
// CTA has published row i+2's max, and the max warps wait for their own epilogue to be done
// with row i before publishing row i+4 (see the comments at the waits).
#pragma once
// (included inside namespace bs)

#ifdef BS_CK_CL
constexpr int CK_CL = BS_CK_CL;           // CTAs per cluster (experiment)
#else
constexpr int CK_CL = 8;                  // CTAs per cluster
#endif
#ifdef BS_CK_NMW
constexpr int CK_NMW = BS_CK_NMW;         // mass warps (experiment)
constexpr int CK_NXW = BS_CK_NXW;         // max warps (experiment)
#else
constexpr int CK_NMW = 8;                 // mass warps: 0..7 (two per SM sub-partition)
constexpr int CK_NXW = 2;                 // max warps: 8..9
#endif
constexpr int CK_NCW = CK_NMW + CK_NXW;
constexpr int CK_PROD = CK_NCW;           // producer warp
constexpr int CK_EPI = CK_NCW + 1;        // epilogue warp
constexpr int CK_CLM = CK_NCW + 2;        // claimer warp (leader CTA)
constexpr int CK_NT = (CK_NCW + 3) * 32;  // 416 threads
#ifdef BS_CK_NB
constexpr int CK_NB = BS_CK_NB;           // slice buffers (experiment)
#else
constexpr int CK_NB = 2;                  // slice buffers
#endif
#ifdef BS_CK_MINB
constexpr int CK_MINB = BS_CK_MINB;       // min CTAs per SM (register budget experiment)
#else
constexpr int CK_MINB = 2;
#endif
#ifdef BS_CK_LA
constexpr int CK_LA = BS_CK_LA;           // claimer look-ahead past the issued copies (experiment)
#else
constexpr int CK_LA = 2;                  // claimer look-ahead past the issued copies
#endif
#ifdef BS_CK_D
constexpr int CK_D = BS_CK_D;             // descriptor / exchange ring depth (experiment)
#else
constexpr int CK_D = 4;                   // descriptor / exchange ring depth
#endif
// ring reuse (see the waits): a peer publishes row i+D only after this CTA's mass warps read
// row i's maxima, which needs D >= 2 x buffers
static_assert(CK_D >= 2 * CK_NB, "exchange ring shallower than twice the slice buffers");
constexpr int CK_TILE = 512;              // elements per tile (16 per lane)
constexpr int CK_BUF_LOCK = 1 << 30;      // slice buffer held by the epilogue (crossing tile)
constexpr int CK_MAXT = 104;              // tiles per slice
constexpr int CK_MAXSL = CK_MAXT * CK_TILE;  // 53248 elements: V <= 425984

struct CkShared {
    uint64_t full[CK_NB], empty[CK_NB];
    uint64_t dfull[CK_D], dempty[CK_D], maxbar[CK_D], sumbar[CK_D], eempty[CK_D];
    RowDesc dq[CK_D];
    uint4 cmax[CK_D][CK_CL];  // per CTA: {slice max bits, bad, greedy index, 0}
    uint4 csum[CK_D][CK_CL];  // per CTA: {slice mass sum lo, hi, mass(d) lo, hi}
    uint4 erec[CK_D];         // mass warps -> epilogue: {m bits, bad, greedy index, 0}
    int mail;  // leader: (rollout << 8 | row) the epilogue found needed next, or -1
    int tma_issued;  // leader: rows whose copy the producer has issued (claimer look-ahead)
    int bufst[CK_NB];  // row (sequence number) a slice buffer holds; | CK_BUF_LOCK while the epilogue reads it
    int plan_b[CK_NMW];  // planning round: rollout per mass warp (-1 dead, -2 none)
    float wmax[CK_NXW];
    uint32_t wbad[CK_NXW];
    int32_t widx[CK_NXW];
    unsigned long long wsum[CK_NMW];
    unsigned long long tsum[CK_D][CK_MAXT];
    unsigned long long stat[STAT_COUNT];
};

__host__ __device__ constexpr size_t ck_smem_bytes(int SL) {
    return ((sizeof(CkShared) + 127) & ~size_t(127)) + (size_t)CK_NB * SL * 2;
}

// ---------------------------------------------------------------- row scheduler
// PLAN.  At kernel start the mass warps of every CTA plan the call's rollouts in parallel
// (one warp per rollout): clamp q (reading L6), validate the draft, reset the rollout's
// completion state, write its record, then publish its claim counter next_row[b] =
// (epoch << 32 | 0) (release; a counter with another epoch reads as "not planned yet").
//
// CLAIM.  Every row claim is atomicAdd(next_row[b]) -> r, kept iff r <= roll_first[b] (the
// lowest deciding row seen, initially q: P:555, rows after the first rejection are not
// needed).  The leader CTA's producer warp picks b:
//   * look-ahead (its buffer still busy): the next rollout of the static cursor (row 0);
//   * buffer free: a warp scan of every rollout's state, best first:
//       READY  row nr-1 completed and accepted: row nr is needed (deepest first),
//       STATIC row 0 not claimed yet,
//       SPEC   row nr-1 still in flight: an idle cluster shortens the chain (shallowest
//              first), so small batches verify all rows of a rollout at once and full
//              batches speculate only while draining;
//     ties rotate by cluster id so concurrent claimers spread over rollouts.
// No queues: the scan only reads, so idle clusters do not contend.  Returns b = -1 once
// every rollout of the call is finalized.
constexpr int SRC_NONE = 0, SRC_READY = 1, SRC_STATIC = 2, SRC_SPEC = 3;

// Static-list order: "hot" rollouts -- a draft and at least CK_HOT_T tokens accepted in the
// previous step (out_acc of the launch before; acceptance runs in streaks while a rollout
// follows its prompt's pool) -- come first, so their likely acceptance chains start early and
// the single-row rollouts fill the end of the launch.  Only the order changes, never a result.
#ifdef BS_HOT_T
constexpr int CK_HOT_T = BS_HOT_T;
#else
constexpr int CK_HOT_T = 2;
#endif
constexpr unsigned long long CK_M21 = (1ull << 21) - 1ull;  // plan word: planned | live | hot, 21 bits each

// Entry idx of the static list: hot rollouts from the front of the live array, the others from
// its back (reversed).
__device__ __forceinline__ const unsigned long long* ck_live_at(const VerifyArgs& a, int idx, int nhot) {
    return a.live + (idx < nhot ? idx : a.n - 1 - (idx - nhot));
}

// Returns 0 if rollout b has no rows, 1 if it is live, 2 if it is live and hot; the caller counts
// and lists it per CTA.
__device__ int ck_plan(const VerifyArgs& a, uint32_t epoch, int b, int lane) {
    const int kp1 = a.k + 1;
    // loads that depend on b only go out with the slot lookup (one round trip)
    const int sl = a.slots[b];
    const int dlen = a.draft_len[b];
    const int prev_acc = (lane == 0) ? a.out_acc[b] : 0;  // the previous step's (read before the reset below)
    const int tk = (lane < a.k) ? a.draft[(int64_t)b * a.k + lane] : 0;
    const int p = a.pos[sl], L = a.max_len[sl];
    int q = -1;
    if (!a.finished[sl] && p < L) q = min(max(dlen, 0), min(a.k, L - p - 1));
    const int t = (lane < q) ? tk : 0;
    if (q > 0 && __any_sync(0xFFFFFFFFu, lane < q && (t < 0 || t >= a.V))) {
        q = -1;
        if (lane == 0) atomicOr(a.dev_err, DEV_BAD_DRAFT);
    }
    if (lane < kp1) {
        if (a.out_norm) a.out_norm[(int64_t)b * kp1 + lane] = 0.f;
        if (a.out_z) a.out_z[(int64_t)b * kp1 + lane] = 0ull;
        if (q < 0) a.out_tokens[(int64_t)b * kp1 + lane] = -1;
    }
    const int d0 = __shfl_sync(0xFFFFFFFFu, t, 0);
    if (lane == 0) {
        RollRec rr;
        rr.q = q;
        rr.slot = sl;
        rr.pos = p;
        rr.tag = (int32_t)epoch;
        rr.uid = a.uid[sl];
        rr.rowno0 = -1;  // row_index is read at claim time (after griddepcontrol.wait)
        rr.d0 = q > 0 ? d0 : -1;
        rr.aligned0 = 0;
        rr.pad[0] = rr.pad[1] = 0;
        a.rrec[b] = rr;
        a.roll_first[b] = q;  // the bonus row q always decides; -1: no rows
        a.roll_state[b] = 0ull;
        if (q < 0) {  // finished / out of length / bad draft: no rows, nothing emitted
            a.out_len[b] = 0;
            a.out_acc[b] = 0;
            if (a.commit) {  // fused commit of an empty step (as commit_kernel): finished,
                // out of length, or a bad draft (an error stop of a live rollout)
                const int f = 1;
                if (f && !a.finished[sl]) a.c_finished[sl] = 1;
                if (a.c_fin_out) a.c_fin_out[b] = f;
            }
        }
        // publish the plan (release: the record and resets above first): claim word =
        // epoch << 32 | (q + 1) << 24 | next row (0)
        st_release_u64(a.next_row + b, ((unsigned long long)epoch << 32) | ((unsigned long long)(q + 1) << 24));
        TRACE(TR_PLANNED, 0, b, 0);
    }
    const bool hot = __shfl_sync(0xFFFFFFFFu, prev_acc >= CK_HOT_T ? 1 : 0, 0) != 0;
    return q < 0 ? 0 : ((q > 0 && hot) ? 2 : 1);
}

// Row r of rollout b as a descriptor (lane-uniform inputs; every lane computes it).
__device__ __forceinline__ RowDesc ck_desc(int b, int j, int q, int d, int pos, unsigned long long uid,
                                           long long rowno, int aligned, int src, int slot) {
    RowDesc r;
    r.b = b;
    r.j = j;
    r.q = q;
    r.d = d;
    r.rowno = rowno;
    r.uid = uid;
    r.position = pos + j;
    r.aligned = aligned;
    r.pad[0] = src;   // claim source (diagnostics)
    r.pad[1] = slot;  // rollout slot (fused commit)
    return r;
}

// Claim the next row of rollout b (lane 0 computes, the warp receives the descriptor).
// Returns false when the claim is not needed (decided below / beyond q / unplanned).
// A row claim in flight: lane 0 holds the claim counter's old value, lane 1 the record and
// roll_first, lanes 2-3 the predicted row's draft token / logits row.  Issued early (the
// loads complete asynchronously), finished when the row is needed.
struct TakeIssue {
    int b = -1, rpred = 0;
    unsigned long long old = 0;
    int rf = -1, q = 0, p = 0, d0 = -1, al0 = 0, dpred = -1, slot = 0;
    unsigned long long u = 0;
    long long rn0 = 0, rnpred = 0;
};

__device__ __forceinline__ TakeIssue ck_take_issue(const VerifyArgs& a, int b, int lane, int rpred) {
    TakeIssue t;
    t.b = b;
    t.rpred = rpred;
    const int kp1 = a.k + 1;
    const RollRec* rp = a.rrec + b;
    if (lane == 0) t.old = atomicAdd(a.next_row + b, 1ull);
    if (lane == 1) {  // L2 reads (published by another SM this launch)
        t.rf = ld_volatile_i32(a.roll_first + b);
        t.q = __ldcg(&rp->q);
        t.slot = __ldcg(&rp->slot);
        t.p = __ldcg(&rp->pos);
        t.u = __ldcg(&rp->uid);
        t.d0 = __ldcg(&rp->d0);
    }
    if (lane == 2 && rpred >= 1 && rpred <= a.k) t.dpred = a.draft[(int64_t)b * a.k + min(rpred, a.k - 1)];
    if (lane == 3 && rpred >= 0 && rpred <= a.k) {
        pdl_wait();  // row_index comes from the previous launch (the claimer starts before it ends)
        t.rnpred = a.row_index ? a.row_index[(int64_t)b * kp1 + rpred] : (int64_t)b * kp1 + rpred;
    }
    return t;
}

__device__ __forceinline__ bool ck_take_finish(const VerifyArgs& a, uint32_t epoch, const TakeIssue& t, int src,
                                               int lane, RowDesc& out) {
    const int kp1 = a.k + 1, b = t.b;
    const unsigned long long old = shfl_u64(t.old, 0);
    const int rf = __shfl_sync(0xFFFFFFFFu, t.rf, 1);
    const int r = (int)(uint32_t)(old & 0xFFFFFFu);
    const bool valid = (uint32_t)(old >> 32) == epoch && r <= rf;
    if (!valid) return false;
    const int q = __shfl_sync(0xFFFFFFFFu, t.q, 1);
    const int sl = __shfl_sync(0xFFFFFFFFu, t.slot, 1);
    const int p = __shfl_sync(0xFFFFFFFFu, t.p, 1);
    const unsigned long long u = shfl_u64(t.u, 1);
    int d = -1, al = 0;
    long long rn = 0;
    if (r == 0) {
        d = __shfl_sync(0xFFFFFFFFu, t.d0, 1);
        if (t.rpred == 0) {
            rn = (long long)shfl_u64((unsigned long long)t.rnpred, 3);
        } else {
            if (lane == 0) {
                pdl_wait();
                rn = a.row_index ? a.row_index[(int64_t)b * kp1] : (int64_t)b * kp1;
            }
            rn = (long long)shfl_u64((unsigned long long)rn, 0);
        }
        al = ((reinterpret_cast<uintptr_t>(a.logits + rn * a.stride) & 15u) == 0) ? 1 : 0;
    } else {
        if (r == t.rpred) {
            d = __shfl_sync(0xFFFFFFFFu, t.dpred, 2);
            rn = (long long)shfl_u64((unsigned long long)t.rnpred, 3);
        } else {
            if (lane == 0) {
                d = (r < q) ? a.draft[(int64_t)b * a.k + r] : -1;
                pdl_wait();
                rn = a.row_index ? a.row_index[(int64_t)b * kp1 + r] : (int64_t)b * kp1 + r;
            }
            d = __shfl_sync(0xFFFFFFFFu, d, 0);
            rn = (long long)shfl_u64((unsigned long long)rn, 0);
        }
        if (r >= q) d = -1;
        al = ((reinterpret_cast<uintptr_t>(a.logits + rn * a.stride) & 15u) == 0) ? 1 : 0;
    }
    out = ck_desc(b, r, q, d, p, u, rn, al, src, sl);
    return true;
}

__device__ __forceinline__ bool ck_take(const VerifyArgs& a, uint32_t epoch, int b, int src, int lane,
                                        int rpred, RowDesc& out) {
    return ck_take_finish(a, epoch, ck_take_issue(a, b, lane, rpred), src, lane, out);
}

// Eager mode: row j of rollout b from the static cursor (each row enumerated exactly once).
__device__ __forceinline__ bool ck_take_row(const VerifyArgs& a, int b, int j, int lane, RowDesc& out) {
    // every load is independent: lanes 0-3 fetch roll_first, the record, the draft token and
    // the logits row in one round trip
    const RollRec* rp = a.rrec + b;
    const int kp1 = a.k + 1;
    int rf = -1, q = 0, p = 0, d0 = -1, al0 = 0, dj = -1, sl = 0;
    unsigned long long u = 0;
    long long rn0 = 0, rnj = 0;
    if (lane == 0) rf = ld_volatile_i32(a.roll_first + b);
    if (lane == 1) {
        q = __ldcg(&rp->q);
        sl = __ldcg(&rp->slot);
        p = __ldcg(&rp->pos);
        u = __ldcg(&rp->uid);
        d0 = __ldcg(&rp->d0);
    }
    if (lane == 2 && j >= 1 && j < a.k) dj = a.draft[(int64_t)b * a.k + j];
    if (lane == 3) {
        pdl_wait();  // row_index comes from the previous launch
        rnj = a.row_index ? a.row_index[(int64_t)b * kp1 + j] : (int64_t)b * kp1 + j;
    }
    rf = __shfl_sync(0xFFFFFFFFu, rf, 0);
    q = __shfl_sync(0xFFFFFFFFu, q, 1);
    if (!(j <= q && j <= rf)) return false;
    p = __shfl_sync(0xFFFFFFFFu, p, 1);
    u = shfl_u64(u, 1);
    int d, al;
    long long rn;
    if (j == 0) d = __shfl_sync(0xFFFFFFFFu, d0, 1);
    else d = (j < q) ? __shfl_sync(0xFFFFFFFFu, dj, 2) : -1;
    rn = (long long)shfl_u64((unsigned long long)rnj, 3);
    al = ((reinterpret_cast<uintptr_t>(a.logits + rn * a.stride) & 15u) == 0) ? 1 : 0;
    sl = __shfl_sync(0xFFFFFFFFu, sl, 1);
    out = ck_desc(b, j, q, d, p, u, rn, al, j == 0 ? SRC_STATIC : SRC_SPEC, sl);
    return true;
}

// Warp scan of every rollout's claim state; returns the best rollout, its class and the
// counter value seen.  Two independent loads per rollout (claim word, state word): one
// round trip per CK_SCAN*32 rollouts.  roll_first is derived: min(q, lowest deciding row).
constexpr int CK_SCAN = 4;
__device__ int ck_scan(const VerifyArgs& a, uint32_t epoch, int lane, int rot, int& src, int& rpred) {
    const int n = a.n;
    unsigned best = 0;
    for (int base = 0; base < n; base += 32 * CK_SCAN) {
        unsigned long long w[CK_SCAN], st[CK_SCAN];
#pragma unroll
        for (int i = 0; i < CK_SCAN; ++i) {
            const int b = base + i * 32 + lane;
            w[i] = (b < n) ? ld_relaxed_u64(a.next_row + b) : 0ull;
            st[i] = (b < n) ? ld_relaxed_u64(a.roll_state + b) : 0ull;
        }
#pragma unroll
        for (int i = 0; i < CK_SCAN; ++i) {
            const int b = base + i * 32 + lane;
            if (b >= n || (uint32_t)(w[i] >> 32) != epoch) continue;  // not planned yet
            const int q = (int)((w[i] >> 24) & 0xFFu) - 1;
            const int nr = (int)(w[i] & 0xFFFFFFu);
            const uint32_t dec = (uint32_t)(st[i] >> 32);
            const int rf = dec ? min(q, __ffs(dec) - 1) : q;
            if (nr > rf) continue;  // every needed row claimed (or no rows)
            unsigned prio, sub;
            if (nr == 0) {
                prio = 2;
                sub = 0;
            } else if (((st[i] >> (nr - 1)) & 1ull) && !((dec >> (nr - 1)) & 1u)) {
                prio = 3;
                sub = (unsigned)nr;  // deepest ready row first
            } else {
                prio = 1;
                sub = 63u - (unsigned)nr;  // shallowest speculation first
            }
            const unsigned rk = (unsigned)(n - 1 - (b - rot + n) % n);  // rotation: b == rot first
            best = max(best, (prio << 30) | (sub << 24) | rk);
        }
    }
    best = __reduce_max_sync(0xFFFFFFFFu, best);
    if (!best) return -1;
    const unsigned pr = best >> 30, sb = (best >> 24) & 63u;
    src = (pr == 3) ? SRC_READY : (pr == 2 ? SRC_STATIC : SRC_SPEC);
    rpred = (pr == 3) ? (int)sb : (pr == 2 ? 0 : 63 - (int)sb);
    const int rk = (int)(best & 0xFFFFFFu);
    return (rot + (n - 1 - rk)) % n;
}

// queues: the caller's buffer is free (any row may be claimed); otherwise look ahead into
// the static cursor only.  Returns b = -2 when the look-ahead finds nothing.
// Producer-side claim state kept across claims (saves round trips once the facts are known).
struct ClaimState {
    int nlive = -1;          // live rollouts (after the plan completed)
    int nhot = 0;            // of which hot (listed first)
    bool eager = false;
    bool static_done = false;  // the static cursor is exhausted
    int spec_b = -1, spec_r = 0;  // chain this cluster just continued: speculate its next row
    int sidx = 0;              // next entry of this cluster's share of the static list (uniform)
    int sh_base = -1;          // share position of the window held in registers (-1: none)
    unsigned long long my_e = 0;  // lane l: live-list entry of share position sh_base + l
    TakeIssue pc;              // pre-issued claim of the next static row (pc.b < 0: none)
    bool post = false;         // ck_post is due after the broadcast
};

// Load a window of 32 entries of this cluster's share of the static list (share position
// p = base + lane is static entry cid + p * ncl) in one round of acquire loads, so the claims'
// record loads are ordered after the planners' publication.  Entries not yet published (the
// plan count precedes the list stores) are polled again.
__device__ __forceinline__ void ck_share_load(const VerifyArgs& a, uint32_t epoch, int lane, ClaimState& cs,
                                              int nstatic, int base) {
    const int cid = (int)(blockIdx.x / CK_CL);
    const int s = cid + (base + lane) * a.ncl;
    bool need = s < nstatic;
    unsigned long long e = 0;
    for (;;) {
        if (need) e = ld_acquire_u64(ck_live_at(a, s % cs.nlive, cs.nhot));
        need = need && (uint32_t)(e >> 32) != epoch;
        if (!__any_sync(0xFFFFFFFFu, need)) break;
        __nanosleep(32);
    }
    cs.sh_base = base;
    cs.my_e = e;
}

// The rollout of static entry cs.sidx, from the register window (loading the next window when
// the share runs past it).
__device__ __forceinline__ int ck_share_get(const VerifyArgs& a, uint32_t epoch, int lane, ClaimState& cs,
                                            int nstatic) {
    const int cid = (int)(blockIdx.x / CK_CL);
    const int k = (cs.sidx - cid) / a.ncl;
    if (cs.sh_base < 0 || k - cs.sh_base >= 32) ck_share_load(a, epoch, lane, cs, nstatic, k);
    return (int)(uint32_t)shfl_u64(cs.my_e, k - cs.sh_base);
}

// Pre-issue the claim of this cluster's next static row: the atomic and loads complete while
// the current row is processed (at a window boundary the next static claim loads the window).
__device__ __forceinline__ void ck_preissue(const VerifyArgs& a, uint32_t epoch, int lane, ClaimState& cs,
                                            int nstatic) {
    if (cs.sidx >= nstatic) return;
    const int cid = (int)(blockIdx.x / CK_CL);
    const int k = (cs.sidx - cid) / a.ncl;
    if (cs.sh_base < 0 || k - cs.sh_base >= 32) return;
    const int b = (int)(uint32_t)shfl_u64(cs.my_e, k - cs.sh_base);
    cs.sidx += a.ncl;
    cs.pc = ck_take_issue(a, b, lane, 0);
}

// Deferred claim bookkeeping, run by the claimer once it has broadcast the row it just claimed
// (nothing is issued between a claim and its broadcast): pre-issue the next static claim.
__device__ __forceinline__ void ck_post(const VerifyArgs& a, uint32_t epoch, int lane, ClaimState& cs) {
    if (!cs.eager && cs.pc.b < 0) ck_preissue(a, epoch, lane, cs, cs.nlive);
}

__device__ __forceinline__ RowDesc ck_claim(const VerifyArgs& a, uint32_t epoch, int lane, bool queues, int rot,
                            ClaimState& cs, int* mail) {
    const int n = a.n;
    uint64_t t_spin0 = 0;
    RowDesc out;
    const int cid = (int)(blockIdx.x / CK_CL);
    if (cs.nlive < 0) {
        // the static list is the live rollouts, compacted by the planners: wait for the plan
        int nl = 0, nh = 0;
        if (lane == 0) {
            const unsigned long long* w = reinterpret_cast<const unsigned long long*>(a.sctl + SC_NLIVE);
            unsigned long long v = ld_acquire_u64(w);
            while ((int)(v >> 42) < n) {
                __nanosleep(32);
                v = ld_acquire_u64(w);
            }
            nl = (int)((v >> 21) & CK_M21);
            nh = (int)(v & CK_M21);
        }
        cs.nlive = __shfl_sync(0xFFFFFFFFu, nl, 0);
        cs.nhot = __shfl_sync(0xFFFFFFFFu, nh, 0);
        // eager when every live row fits in flight at once (two per cluster): the static
        // list then enumerates every row, j-major, and a cluster leaves once it is exhausted
        cs.eager = a.eager_ok == 2 || (a.eager_ok && (long long)cs.nlive * (a.k + 1) <= (long long)CK_NB * a.ncl);
        cs.sidx = cid;
        cs.sh_base = -1;
    }
    const int nlive = cs.nlive;
    const bool eager = cs.eager;
    const int nstatic = eager ? nlive * (a.k + 1) : nlive;
    for (int spin = 0;; ++spin) {
        // 1. this cluster's own epilogue accepted row j of rollout b: row j+1 is needed and
        //    the chain stays here (no scan)
        if (!eager) {
            int mb = -1;
            if (lane == 0) mb = atomicExch(mail, -1);  // read and clear in one shared atomic
            mb = __shfl_sync(0xFFFFFFFFu, mb, 0);
            if (mb >= 0) {
                if (ck_take(a, epoch, mb >> 8, SRC_READY, lane, mb & 0xFF, out)) {
                    cs.spec_b = mb >> 8;  // next claim: the chain's following row, speculatively
                    cs.spec_r = out.j + 1;
                    return out;
                }
                continue;
            }
        }
        // 2. this cluster's share of the static list (entries cid, cid + ncl, ...: no shared
        //    cursor); the share is held in registers, 32 entries per window, and the next
        //    static claim is pre-issued, so a static claim costs no dependent round trip.
        //    Other clusters' unclaimed rows 0 are stolen by the scan once a share is done.
        // 2a. the static row whose claim was pre-issued by the previous static claim
        if (!eager && cs.pc.b >= 0) {
            const TakeIssue t = cs.pc;
            cs.pc.b = -1;
            if (ck_take_finish(a, epoch, t, SRC_STATIC, lane, out)) {
                cs.post = true;
                return out;
            }
            ck_post(a, epoch, lane, cs);
            continue;
        }
        int b = -1, j = 0;
        if (!cs.static_done) {
            if (cs.sidx < nstatic) {
                b = ck_share_get(a, epoch, lane, cs, nstatic);
                j = cs.sidx / nlive;
                cs.sidx += a.ncl;
            }
            if (b < 0) cs.static_done = true;
        }
        if (b >= 0) {
            const bool ok = eager ? ck_take_row(a, b, j, lane, out) : ck_take(a, epoch, b, SRC_STATIC, lane, 0, out);
            if (ok) {
                cs.post = true;
                return out;
            }
            ck_post(a, epoch, lane, cs);
            continue;
        }
        // no certain work left in the static list: speculate the chain just continued here
        // (its second buffer would idle otherwise; a dead row stops early)
        if (cs.spec_b >= 0) {
            const int sb = cs.spec_b, sr = cs.spec_r;
            cs.spec_b = -1;
            if (sr <= a.k && ck_take(a, epoch, sb, SRC_SPEC, lane, sr, out)) return out;
        }
        if (eager) break;  // every row claimed: nothing left for this cluster
        {
            int src = SRC_NONE, rpred = 0;
            b = ck_scan(a, epoch, lane, rot, src, rpred);
            if (lane == 0) TRACE(TR_ITER, spin, b, src);
            if (b >= 0) {
                if (ck_take(a, epoch, b, src, lane, rpred, out)) return out;
                continue;
            }
        }
        // nothing claimable now: done, or wait for rows to complete.  The decision is
        // lane 0's (a per-lane read of a changing word could split the warp)
        int done = 0;
        if (lane == 0) done = ((int)ld_relaxed_u32(a.sctl + SC_DONE) >= n) ? 1 : 0;
        if (__shfl_sync(0xFFFFFFFFu, done, 0)) {
            if (lane == 0) TRACE(TR_SPINS, spin, 0, 0);
            break;
        }
        if (!queues) {  // static cursor exhausted: the caller retries once its buffer is free
            out.b = -2;
            return out;
        }
        __nanosleep(64);
        if (spin == 0) t_spin0 = globaltimer_ns();
        if ((spin & 1023) == 1023 && lane == 0 && globaltimer_ns() - t_spin0 > 1500000000ull) {
            // 1.5 s without claimable work: protocol bug
#ifdef BS_TRACE
            printf("bs sched stall: block %d done %u n %d\n", (int)blockIdx.x, a.sctl[SC_DONE], n);
#endif
            __trap();
        }
    }
    out.b = -1;
    return out;
}

// Masses of 16 consecutive logits (two 16-byte vectors), elements >= nvalid or == excl
// zeroed (indices relative to the first element).
__device__ __forceinline__ void ck_mass16(const uint4 v0, const uint4 v1, const MassParams& mp,
                                          int e0, int nvalid, int excl, uint64_t mm[16]) {
    mass8_masked(v0, mp, e0, nvalid, excl, mm);
    mass8_masked(v1, mp, e0 + 8, nvalid, excl, mm + 8);
}

__global__ void __cluster_dims__(CK_CL, 1, 1) __launch_bounds__(CK_NT, CK_MINB)
    verify_cluster_kernel(const VerifyArgs a, int SL) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(128) uint8_t ck_smem[];
    CkShared& sh = *reinterpret_cast<CkShared*>(ck_smem);
    uint16_t* bufs = reinterpret_cast<uint16_t*>(ck_smem + ((sizeof(CkShared) + 127) & ~size_t(127)));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rank = (int)cluster.block_rank();
    const int V = a.V;
    const int e_lo = rank * SL;
    const int len = max(0, min(SL, V - e_lo));
    const int ntile = (len + CK_TILE - 1) / CK_TILE;
    if (tid == 0) {
        for (int i = 0; i < CK_NB; ++i) {
            mbar_init(&sh.full[i], 1);
            mbar_init(&sh.empty[i], CK_NMW);  // the mass warps are the buffer's last readers
        }
        for (int i = 0; i < CK_D; ++i) {
            mbar_init(&sh.dfull[i], 1);
            mbar_init(&sh.dempty[i], CK_CL);
            mbar_init(&sh.maxbar[i], 1);
            mbar_init(&sh.sumbar[i], 1);
            mbar_init(&sh.eempty[i], 1);
        }
        fence_mbar_init();
    }
    for (int i = tid; i < STAT_COUNT; i += CK_NT) sh.stat[i] = 0ull;
    if (tid == 0) {
        sh.mail = -1;
        sh.tma_issued = 0;
        for (int x = 0; x < CK_NB; ++x) sh.bufst[x] = -1;
    }
#ifdef BS_TRACE
    if (tid == 0) {
        s_trace_n = 0;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        TRACE(TR_START, 0, (int)smid, 0);
    }
#endif
    // every CTA's barriers exist before any remote operation: the mbarrier inits are published by
    // fence.mbarrier_init.release.cluster above, so a relaxed cluster arrive suffices (no full
    // fence); the CTA's own shared-memory initialisation is ordered by the CTA barrier
    __syncthreads();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    // Without the caller's early-plan promise (bsx_set_early_plan) everything waits for the
    // previous kernel first: only griddepcontrol.wait makes its writes visible.
    if (!a.early_plan) pdl_wait();
    // With it, the plan runs before griddepcontrol.wait, overlapping the kernel launched just before
    // this one (the model forward / target rows): its inputs (slots, drafts, positions,
    // lengths, uids) come from launches at least two back (the lookup triggers its dependents
    // only after its stores), and it reads no logits and no row_index.  The previous verify
    // launch is complete (the lookup waited for it), so the scheduler words are reset.
    const uint32_t epoch = ld_relaxed_u32(a.sctl + SC_EPOCH);
    // No early launch_dependents: the next launch may plan before its own wait, so it must
    // not start before this one's scheduler state, plan records and fused commit are final
    // (the implicit trigger at exit).
    // The claimer waits only before its row_index loads (ck_take_*): its claims' other
    // inputs are this launch's plan.
    if (warp >= CK_NMW && warp != CK_CLM) pdl_wait();
    if (tid == 0) TRACE(TR_GO, 0, 0, 0);
    if (warp < CK_NMW) {
        // plan the call's rollouts, one warp each, in rounds over the grid; per round one atomic
        // per CTA counts its planned rollouts (high half of the packed word) and reserves its
        // live-list slots (low half), so the plan's completion count is not one hot word
        for (int base = (int)blockIdx.x * CK_NMW; base < a.n; base += (int)gridDim.x * CK_NMW) {
            const int b = base + warp;
            const int live = (b < a.n) ? ck_plan(a, epoch, b, lane) : 0;
            if (lane == 0) sh.plan_b[warp] = (b < a.n) ? (live ? (b | (live == 2 ? (1 << 30) : 0)) : -1) : -2;
            named_bar(3, CK_NMW * 32);
            if (warp == 0 && lane == 0) {
                int np = 0, nl = 0, nh = 0;
                for (int w = 0; w < CK_NMW; ++w) {
                    np += sh.plan_b[w] != -2;
                    nl += sh.plan_b[w] >= 0;
                    nh += sh.plan_b[w] >= (1 << 30);
                }
                // rollouts without rows are done (one termination-count atomic per CTA round)
                if (np > nl) atomicAdd(a.sctl + SC_DONE, (unsigned)(np - nl));
                // planned << 42 | live << 21 | hot: counts and list slots in one atomic
                const unsigned long long cnt =
                    atomicAdd(reinterpret_cast<unsigned long long*>(a.sctl + SC_NLIVE),
                              ((unsigned long long)np << 42) | ((unsigned long long)nl << 21) | (unsigned long long)nh);
                unsigned hs = (unsigned)(cnt & CK_M21);
                unsigned cs = (unsigned)((cnt >> 21) & CK_M21) - hs;
                for (int w = 0; w < CK_NMW; ++w) {
                    const int pb = sh.plan_b[w];
                    if (pb < 0) continue;
                    const int bb = pb & ((1 << 30) - 1);
                    unsigned long long* dst = (pb >= (1 << 30)) ? a.live + hs++ : a.live + (a.n - 1 - (int)cs++);
                    st_release_u64(dst, ((unsigned long long)epoch << 32) | (uint32_t)bb);
                }
            }
            named_bar(3, CK_NMW * 32);  // plan_b reusable
        }
        pdl_wait();
        if (a.lookup) {
            // fused lookup for the rollouts without rows (finished, out of length, bad draft):
            // their (empty) commit was the plan's; the finalizing epilogue warps look up the
            // others.  After the wait: the launch before this one (the target) reads the drafts.
            __syncwarp();
            for (int base = (int)blockIdx.x * CK_NMW; base < a.n; base += (int)gridDim.x * CK_NMW) {
                const int b = base + warp;
                if (b >= a.n) break;
                const int q = __shfl_sync(0xFFFFFFFFu, lane == 0 ? a.rrec[b].q : 0, 0);  // own store
                if (q >= 0) continue;
                const LookupArgs& lk = a.lk;
                const int sl = a.slots[b];
                const int M = lk.M;
                const int tr = (lane < M) ? lk.tail[(int64_t)sl * M + (M - 1 - lane)] : -1;
                const IndexDesc x = *lk.desc;
                lookup_rollout(lk, x, b, lk.ctx_len[sl], lk.prompt[sl], lk.pos[sl], lk.max_len[sl],
                               lk.finished[sl] != 0, tr, lane, x.step != *lk.cur_step);
            }
        }
    }

    if (warp == CK_CLM) {
        // ================================================================ claimer (leader)
        // Claims rows up to two ahead of the producer's copy issue and broadcasts each
        // descriptor to the 8 CTAs with 24 lanes (8 CTAs x 3 x 16 bytes).  A claim is a few
        // dependent round trips (~1.5 us each under full HBM load); in its own warp it never
        // delays a copy.  It blocks (spins for work) only when every row it claimed has had
        // its copy issued: a row waiting for a copy may be the one whose completion creates
        // the work.
        if (rank == 0) {
            const int ncl = (int)(gridDim.x / CK_CL);
            const int rot = (int)(((long long)(blockIdx.x / CK_CL) * a.n) / max(1, ncl));
            ClaimState cst;
            for (int r = 0;;) {
                int issued = 0;
                if (lane == 0) issued = atomicOr(&sh.tma_issued, 0);  // (an atomic: no shared-memory race)
                issued = __shfl_sync(0xFFFFFFFFu, issued, 0);
                if (r > issued + CK_LA) {  // far enough ahead
                    __nanosleep(128);
                    continue;
                }
                const int s = r % CK_D;
                if (lane == 0) TRACE(TR_LOOP, r, 0, 0);
                // every CTA's epilogue is done with row r-4 (the slot's previous use)
                if (r >= CK_D) mbar_wait_cluster(&sh.dempty[s], ((r / CK_D) - 1) & 1);
                if (lane == 0) TRACE(TR_CLAIM0, r, 0, 0);
                const RowDesc nd = ck_claim(a, epoch, lane, r <= issued, rot, cst, &sh.mail);
                if (nd.b == -2) {  // nothing claimable now, and rows are still being copied
                    __nanosleep(128);
                    continue;
                }
                if (lane == 0) TRACE(TR_CLAIM1, r | (nd.b >= 0 ? nd.pad[0] << 12 : 0), nd.b, nd.j);
                uint32_t w[12];
                memcpy(w, &nd, sizeof(w));
                for (int x = lane; x < 3 * CK_CL; x += 32) {
                    const int part = x % 3;
                    uint4 v = make_uint4(w[0], w[1], w[2], w[3]);
                    if (part == 1) v = make_uint4(w[4], w[5], w[6], w[7]);
                    if (part == 2) v = make_uint4(w[8], w[9], w[10], w[11]);
                    st_async_v4(reinterpret_cast<uint4*>(&sh.dq[s]) + part, v, &sh.dfull[s], (uint32_t)(x / 3));
                }
                if (lane == 0) TRACE(TR_BCAST, r, (int)(w[4] ^ w[5] ^ w[6] ^ w[7]) & 0x7FFF, 0);
                ++r;
                if (nd.b < 0) break;  // END broadcast: nothing more is claimed
                if (cst.post) {
                    cst.post = false;
                    ck_post(a, epoch, lane, cst);
                }
                if (lane == 0) TRACE(TR_POST, r, 0, 0);
            }
        }
    } else if (warp == CK_PROD) {
        // ================================================================ producer
        // Every CTA: bulk-copies (TMA) its slice of each row into one of two buffers.
        if (lane == 0) mbar_arrive_expect_tx(&sh.dfull[0], (uint32_t)sizeof(RowDesc));
        for (int i = 0;; ++i) {
            const int s = i % CK_D, bi = i % CK_NB;
            // arm the descriptor slot for row i (its use by row i-4 completed: this warp
            // waited on it); the leader's bytes may already have arrived
            if (i > 0 && lane == 0) mbar_arrive_expect_tx(&sh.dfull[s], (uint32_t)sizeof(RowDesc));
            mbar_wait(&sh.dfull[s], (i / CK_D) & 1);
            const RowDesc dsc = sh.dq[s];
            if (dsc.b < 0) break;
            if (lane == 0) TRACE(TR_PDESC, i, dsc.b, dsc.j);
            // the slice buffer is free once the mass warps are done with row i-2
            if (i >= CK_NB) mbar_wait(&sh.empty[bi], ((i / CK_NB) - 1) & 1);
            if (lane == 0) {
                // take the buffer over from row i-2 (wait while that row's epilogue reads its
                // crossing tile from it)
                const int prev = (i >= CK_NB) ? i - CK_NB : -1;
                while (atomicCAS(&sh.bufst[bi], prev, i) != prev) __nanosleep(32);
                uint16_t* buf = bufs + (size_t)bi * SL;
                const uint16_t* src = a.logits + dsc.rowno * a.stride + e_lo;
                const int nb = dsc.aligned ? (len & ~7) : 0;  // 16-byte multiple
                for (int e = nb; e < len; ++e) buf[e] = src[e];  // ragged end / unaligned row
                TRACE(TR_TMA, i, dsc.b, dsc.j);
                if (nb) {
                    fence_proxy_async_smem();
                    mbar_arrive_expect_tx(&sh.full[bi], (uint32_t)nb * 2u);
                    // streamed once: evict-first keeps the draft index and pools L2-resident
                    bulk_g2s(buf, src, (uint32_t)nb * 2u, &sh.full[bi], policy_evict_first());
                } else {
                    mbar_arrive(&sh.full[bi]);
                }
                if (rank == 0) atomicExch(&sh.tma_issued, i + 1);
            }
        }
    } else if (warp == CK_EPI) {
        // ================================================================ epilogue
        MassParams mp;
        mp.c = a.c;
        mp.clampv = -(float)(a.S + 2);
        mp.magic = 12582912.0f + (float)a.S;
        for (int i = 0;; ++i) {
            const int s = i % CK_D;
            mbar_wait(&sh.dfull[s], (i / CK_D) & 1);
            const RowDesc dsc = sh.dq[s];
            if (dsc.b < 0) break;
            // fused commit: the rollout's state, fetched while this row's sums arrive (only the
            // finalizing row uses it; nothing else writes it during the launch)
            CommitPre cp;
            if (a.commit) cp = commit_prefetch(a, dsc.pad[1], lane);
            // issued with the descriptor, used after the sums arrive (no round trip after them)
            const int rf_early = (lane == 0) ? ld_volatile_i32(a.roll_first + dsc.b) : 0;
            // the rollout's draft tokens, for its finalize (d_1..d_F); read before this launch's
            // fused lookup can rewrite them (that happens only after the rollout's one finalize)
            const int32_t dpf = (lane < dsc.q) ? a.draft[(int64_t)dsc.b * a.k + lane] : -1;
            mbar_wait(&sh.sumbar[s], (i / CK_D) & 1);
            const int b = dsc.b, j = dsc.j, q = dsc.q, d = dsc.d;
            if (lane == 0) TRACE(TR_EPI0, i, b, j);
            // a row above an already-decided row is not needed: no completion.  Dead
            // is monotone; the view is taken when the descriptor arrives, so a row that became
            // dead later (its max warps may have skipped it) can still be completed here: its
            // record lies above the deciding row F and the finalize reads rows 0..F only, so
            // such a completion changes nothing.
            const bool dead = __shfl_sync(0xFFFFFFFFu, lane == 0 ? (rf_early < j ? 1 : 0) : 0, 0);
            if (dead) {
                __syncwarp();
                if (lane == 0) {
                    TRACE(TR_EPI1, i, dsc.b, dsc.j);
                    mbar_arrive(&sh.eempty[s]);
                    mbar_arrive_remote(&sh.dempty[s], 0u);
                }
                continue;
            }
            if (lane == 0) TRACE(TR_EX1, i, dsc.b, dsc.j);
            const uint4 er = sh.erec[s];  // the cluster max of row i (local record)
            const float m = __uint_as_float(er.x);
            const uint32_t bad = er.y;
            uint64_t Z = 0, md = 0;
#pragma unroll
            for (int r = 0; r < CK_CL; ++r) {
                const uint4 cs = sh.csum[s][r];
                Z += (uint64_t)cs.x | ((uint64_t)cs.y << 32);
                md += (uint64_t)cs.z | ((uint64_t)cs.w << 32);
            }
            uint32_t err = 0;
            if (bad) err |= DEV_BAD_LOGIT;
            else if (m == -INFINITY) err |= DEV_ALL_NEGINF;
            else if (a.T > 0.f && !(fabsf(__fmul_rn(m, a.c)) < 16777216.0f)) err |= DEV_RANGE;
            // the row's result (recorded by one CTA's epilogue warp: the CTA that owns the
            // sampled token, else a rank that rotates with (b, j), so the completions of accepted
            // rows -- a few dependent round trips each -- spread over the cluster's 8 epilogue
            // warps instead of queueing on one)
            const int rec_rank = (int)((unsigned)(3 * b + j) % (unsigned)CK_CL);
            bool rec = false;
            int c_status = ST_DECIDED, c_cand = -1;
            unsigned long long c_z = 0ull;
            float c_norm = 0.f;
            if (err) {  // R0: reported at finalize only if Alg. 1 needs this row
                rec = rank == rec_rank;
                c_status = ST_ERR;
                c_cand = (int)err;
            } else if (a.T == 0.f) {  // greedy (R1): lowest index attaining m
                const int g = (int)er.z;
                const bool acc = j < q && d == g;
                rec = rank == rec_rank;
                c_status = acc ? ((a.eos >= 0 && d == a.eos) ? ST_EOS : ST_CONT) : ST_DECIDED;
                c_cand = g;
                c_z = 1ull;
                c_norm = 1.f;
            } else {
                const float norm = (float)ldexp((double)Z, -a.S);
                bool acc = false;
                if (j < q) acc = uniform_floor(row_draw(a, dsc, PURPOSE_ACCEPT), Z) < md;
                const int status = acc ? ((a.eos >= 0 && d == a.eos) ? ST_EOS : ST_CONT) : ST_DECIDED;
                if (status != ST_DECIDED) {
                    rec = rank == rec_rank;
                    c_status = status;
                    c_z = Z;
                    c_norm = norm;
                } else {
                    // residual (d excluded) or bonus sample (R8): inverse CDF in ascending id
                    const int excl = (j < q) ? d : -1;
                    const uint64_t U =
                        uniform_floor(row_draw(a, dsc, PURPOSE_SAMPLE), Z - ((j < q) ? md : 0ull));
                    const int exr = (excl >= 0) ? excl / SL : -1;
                    int rc = -1;
                    uint64_t cum = 0, ul = 0;
#pragma unroll
                    for (int r = 0; r < CK_CL; ++r) {
                        const uint64_t cs = ((uint64_t)sh.csum[s][r].x | ((uint64_t)sh.csum[s][r].y << 32)) -
                                            ((r == exr) ? md : 0ull);
                        if (rc < 0 && U < cum + cs) {
                            rc = r;
                            ul = U - cum;
                        }
                        cum += cs;
                    }
                    if (lane == 0) TRACE(TR_EX2, i, rc, dsc.j);
                    if (rc == rank) {
                        // crossing tile of this slice (the excluded token's mass off its tile)
                        const int excl_l = excl - e_lo;  // slice-relative (may be out of range)
                        const int ex_t = (excl_l >= 0 && excl_l < len) ? excl_l / CK_TILE : -1;
                        const int per = (ntile + 31) / 32;
                        const int i0 = min(ntile, lane * per), i1 = min(ntile, i0 + per);
                        uint64_t ls = 0;
                        for (int t = i0; t < i1; ++t) ls += sh.tsum[s][t] - ((t == ex_t) ? md : 0ull);
                        const uint64_t incl = warp_incl_scan_u64(ls, lane);
                        const unsigned hit = __ballot_sync(0xFFFFFFFFu, ul < incl);
                        const int L = hit ? (__ffs(hit) - 1) : 31;
                        int xt = 0;
                        uint64_t ut = 0;
                        if (lane == L) {
                            uint64_t c2 = incl - ls;
                            for (int t = i0; t < i1; ++t) {
                                const uint64_t ts = sh.tsum[s][t] - ((t == ex_t) ? md : 0ull);
                                if (ul < c2 + ts) {
                                    xt = t;
                                    ut = ul - c2;
                                    break;
                                }
                                c2 += ts;
                            }
                        }
                        xt = __shfl_sync(0xFFFFFFFFu, xt, L);
                        ut = shfl_u64(ut, L);
                        // the crossing tile: lane l owns its 16 consecutive elements; from the
                        // slice buffer while no later row has taken it over (locked meanwhile),
                        // else re-read from L2 / HBM
                        const int bi = i % CK_NB;
                        int own = 0;
                        if (lane == 0) own = atomicCAS(&sh.bufst[bi], i, i | CK_BUF_LOCK) == i;
                        own = __shfl_sync(0xFFFFFFFFu, own, 0);
                        const uint16_t* rowp = a.logits + dsc.rowno * a.stride + e_lo;
                        const int e0 = xt * CK_TILE + lane * 16;
                        uint4 v0, v1;
                        if (own) {
                            const uint16_t* bp = bufs + (size_t)bi * SL;
                            if (e0 + 16 <= len) {
                                v0 = lds128(bp + e0);
                                v1 = lds128(bp + e0 + 8);
                            } else {
                                uint16_t t16[16];
                                for (int x = 0; x < 16; ++x) t16[x] = (e0 + x < len) ? bp[e0 + x] : (uint16_t)0xFF80u;
                                v0 = make_uint4(t16[0] | ((uint32_t)t16[1] << 16), t16[2] | ((uint32_t)t16[3] << 16),
                                                t16[4] | ((uint32_t)t16[5] << 16), t16[6] | ((uint32_t)t16[7] << 16));
                                v1 = make_uint4(t16[8] | ((uint32_t)t16[9] << 16), t16[10] | ((uint32_t)t16[11] << 16),
                                                t16[12] | ((uint32_t)t16[13] << 16), t16[14] | ((uint32_t)t16[15] << 16));
                            }
                        } else if (dsc.aligned && e0 + 16 <= len) {
                            v0 = __ldcg(reinterpret_cast<const uint4*>(rowp + e0));
                            v1 = __ldcg(reinterpret_cast<const uint4*>(rowp + e0 + 8));
                        } else {
                            uint16_t t16[16];
                            for (int x = 0; x < 16; ++x) t16[x] = (e0 + x < len) ? rowp[e0 + x] : (uint16_t)0xFF80u;
                            v0 = make_uint4(t16[0] | ((uint32_t)t16[1] << 16), t16[2] | ((uint32_t)t16[3] << 16),
                                            t16[4] | ((uint32_t)t16[5] << 16), t16[6] | ((uint32_t)t16[7] << 16));
                            v1 = make_uint4(t16[8] | ((uint32_t)t16[9] << 16), t16[10] | ((uint32_t)t16[11] << 16),
                                            t16[12] | ((uint32_t)t16[13] << 16), t16[14] | ((uint32_t)t16[15] << 16));
                        }
                        mp.nmc = -__fmul_rn(m, a.c);
                        uint64_t mm[16];
                        ck_mass16(v0, v1, mp, e0, len, excl_l, mm);
                        if (own) {  // every lane has consumed its tile registers: hand the buffer back
                            __syncwarp();
                            if (lane == 0) atomicExch(&sh.bufst[bi], i);
                        }
                        uint64_t sl = 0;
#pragma unroll
                        for (int x = 0; x < 16; ++x) sl += mm[x];
                        const uint64_t inc2 = warp_incl_scan_u64(sl, lane);
                        const unsigned hit2 = __ballot_sync(0xFFFFFFFFu, ut < inc2);
                        const int L2 = hit2 ? (__ffs(hit2) - 1) : 31;
                        int tok = -1;
                        if (lane == L2) {
                            uint64_t c3 = inc2 - sl;
                            for (int x = 0; x < 16; ++x) {
                                c3 += mm[x];
                                if (c3 > ut) {
                                    tok = e_lo + e0 + x;
                                    break;
                                }
                            }
                        }
                        tok = __shfl_sync(0xFFFFFFFFu, tok, L2);
                        rec = true;
                        c_cand = tok;
                        c_z = Z;
                        c_norm = norm;
                    }
                }
            }
            if (lane == 0) TRACE(TR_EX3, i, dsc.b, dsc.j);
            // The row's result is in registers: an accepted row posts its successor to this
            // cluster's mailbox (row j+1 is needed: the chain continues here) and the row's
            // slot is handed back before the completion protocol's round trips, so neither the
            // chain nor the claimer (which reuses the slot four rows later) waits for them.
            __syncwarp();
            if (lane == 0) {
                if (rec && c_status == ST_CONT)  // the leader's claimer reads the mailbox
                    atomicExch(cluster.map_shared_rank(&sh.mail, 0), (b << 8) | (j + 1));
                TRACE(TR_EPI1, i, dsc.b, dsc.j);
                mbar_arrive(&sh.eempty[s]);             // tile sums / sum slot of row i free
                mbar_arrive_remote(&sh.dempty[s], 0u);  // descriptor slot of row i free
            }
            if (rec) {  // warp-uniform
                if (lane == 0) sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                int no = 0;
                int32_t ot = -1;
                const bool fz = complete_row_warp(a, sh.stat, b, j, q, c_status, c_cand, c_z, c_norm, lane, no, ot, dpf);
                if (a.commit && fz) commit_rollout_warp(a, b, lane, cp, no, ot);
            }
        }
    } else if (warp >= CK_NMW) {
        // ================================================================ max warps
        const int xw = warp - CK_NMW;
        for (int i = 0;; ++i) {
            const int s = i % CK_D, bi = i % CK_NB;
            mbar_wait(&sh.dfull[s], (i / CK_D) & 1);
            if (sh.dq[s].b < 0) break;
            // dead row (a lower row of its rollout decided): skip the work; the load is
            // issued now and used after the data wait
            const int rfx = ld_volatile_i32(a.roll_first + sh.dq[s].b);
            const int jx = sh.dq[s].j;
            // this CTA's epilogue is done with row i-4 (sum slot, tile sums): every peer's
            // row-i publish lands on completed phases of this CTA's rings
            if (i >= CK_D) mbar_wait(&sh.eempty[s], ((i / CK_D) - 1) & 1);
            if (a.rs_key) {
                // the LM-head epilogue already reduced this row (R0 / R1): publish its maximum,
                // lowest argmax and NaN / +inf flag without reading the slice
                if (xw == 0) {
                    const long long rn = sh.dq[s].rowno;
                    const unsigned long long kv = __ldg(a.rs_key + rn);
                    const uint32_t kb = (uint32_t)(kv >> 32);
                    const uint32_t bits = (kb & 0x8000u) ? (kb & 0x7FFFu) : (~kb & 0xFFFFu);
                    const float sm = __uint_as_float(bits << 16);
                    const uint32_t sb = (__ldg(a.rs_bad + rn) != 0u || kv == 0ull) ? 1u : 0u;
                    const uint32_t sidx = (a.T == 0.f) ? (uint32_t)(0xFFFFFFFFull - (kv & 0xFFFFFFFFull)) : 0x7FFFFFFFu;
                    if (lane == 0) mbar_arrive_expect_tx(&sh.maxbar[s], (uint32_t)(CK_CL * 16));
                    __syncwarp();
                    if (lane < CK_CL)
                        st_async_v4(&sh.cmax[s][rank], make_uint4(__float_as_uint(sm), sb, sidx, 0u), &sh.maxbar[s],
                                    (uint32_t)lane);
                }
                continue;
            }
            mbar_wait(&sh.full[bi], (i / CK_NB) & 1);
            const bool xdead = __shfl_sync(0xFFFFFFFFu, rfx < jx ? 1 : 0, 0) != 0;
            if (xw == 0 && lane == 0) TRACE(TR_MAX0, i, 0, 0);
            const uint16_t* buf = bufs + (size_t)bi * SL;
            uint32_t mx = 0xFF80FF80u, mx1 = 0xFF80FF80u;
            const int nfull = xdead ? 0 : len / CK_TILE;  // whole tiles
            int t = xdead ? ntile : xw;
            for (; t + 3 * CK_NXW < nfull; t += 4 * CK_NXW) {  // 4 tiles per step: 8 loads in flight
                uint4 v[8];
#pragma unroll
                for (int u2 = 0; u2 < 4; ++u2) {
                    // lane l: elements 8l.. and 256+8l.. of the tile (conflict-free 16-byte loads)
                    v[2 * u2] = lds128(buf + (t + u2 * CK_NXW) * CK_TILE + lane * 8);
                    v[2 * u2 + 1] = lds128(buf + (t + u2 * CK_NXW) * CK_TILE + CK_TILE / 2 + lane * 8);
                }
#pragma unroll
                for (int u2 = 0; u2 < 8; u2 += 2) {
                    mx = hmax2_nan_u32(mx, hmax2_nan_u32(hmax2_nan_u32(v[u2].x, v[u2].y), hmax2_nan_u32(v[u2].z, v[u2].w)));
                    mx1 = hmax2_nan_u32(mx1, hmax2_nan_u32(hmax2_nan_u32(v[u2 + 1].x, v[u2 + 1].y),
                                                           hmax2_nan_u32(v[u2 + 1].z, v[u2 + 1].w)));
                }
            }
            for (; t < ntile; t += CK_NXW) {
                const int e0 = t * CK_TILE + lane * 16;
                if (t < nfull) {
                    const uint4 v0 = lds128(buf + t * CK_TILE + lane * 8);
                    const uint4 v1 = lds128(buf + t * CK_TILE + CK_TILE / 2 + lane * 8);
                    mx = hmax2_nan_u32(mx, hmax2_nan_u32(hmax2_nan_u32(v0.x, v0.y), hmax2_nan_u32(v0.z, v0.w)));
                    mx1 = hmax2_nan_u32(mx1, hmax2_nan_u32(hmax2_nan_u32(v1.x, v1.y), hmax2_nan_u32(v1.z, v1.w)));
                } else {
                    for (int x = 0; x < 16; ++x)
                        if (e0 + x < len) mx = hmax2_nan_u32(mx, (uint32_t)buf[e0 + x] | 0xFF800000u);
                }
            }
            mx = hmax2_nan_u32(mx, mx1);
            const float lo = bf16lo(mx), hi = bf16hi(mx);
            uint32_t bad = (isnan(lo) || isnan(hi) || lo == INFINITY || hi == INFINITY) ? 1u : 0u;
            float fm = fmaxf(lo, hi);
#pragma unroll
            for (int k2 = 16; k2; k2 >>= 1) fm = fmaxf(fm, __shfl_xor_sync(0xFFFFFFFFu, fm, k2));
            bad = __any_sync(0xFFFFFFFFu, bad) ? 1u : 0u;
            if (lane == 0) {
                sh.wmax[xw] = fm;
                sh.wbad[xw] = bad;
            }
            named_bar(2, CK_NXW * 32);
            float sm = -INFINITY;
            uint32_t sb = 0;
#pragma unroll
            for (int w = 0; w < CK_NXW; ++w) {
                sm = fmaxf(sm, sh.wmax[w]);
                sb |= sh.wbad[w];
            }
            int sidx = 0x7FFFFFFF;
            if (a.T == 0.f && sm > -INFINITY && !sb) {  // greedy: lowest index attaining sm
                int fi = 0x7FFFFFFF;
                for (int t = xw; t < ntile && fi == 0x7FFFFFFF; t += CK_NXW) {
                    const int e0 = t * CK_TILE + lane * 16;
                    int li = 0x7FFFFFFF;
                    for (int x = 15; x >= 0; --x)
                        if (e0 + x < len && __uint_as_float((uint32_t)buf[e0 + x] << 16) == sm) li = e0 + x;
#pragma unroll
                    for (int k2 = 16; k2; k2 >>= 1) li = min(li, __shfl_xor_sync(0xFFFFFFFFu, li, k2));
                    fi = li;  // a warp's tiles ascend: its first hit is its lowest
                }
                if (lane == 0) sh.widx[xw] = fi;
                named_bar(2, CK_NXW * 32);
#pragma unroll
                for (int w = 0; w < CK_NXW; ++w) sidx = min(sidx, sh.widx[w]);
                if (sidx != 0x7FFFFFFF) sidx += e_lo;
            }
            if (xw == 0) {
                // arm row i's max slot (its row i-4 phase completed: the mass warps waited on
                // it before freeing the buffer this row now occupies), then one lane per CTA
                if (lane == 0) mbar_arrive_expect_tx(&sh.maxbar[s], (uint32_t)(CK_CL * 16));
                __syncwarp();
                if (lane < CK_CL)
                    st_async_v4(&sh.cmax[s][rank], make_uint4(__float_as_uint(sm), sb, (uint32_t)sidx, 0u),
                                &sh.maxbar[s], (uint32_t)lane);
                if (lane == 0) TRACE(TR_MAX1, i, 0, 0);
            }
            named_bar(2, CK_NXW * 32);  // wmax / widx reusable
        }
    } else {
        // ================================================================ mass warps
        MassParams mp;
        mp.c = a.c;
        mp.clampv = -(float)(a.S + 2);
        mp.magic = 12582912.0f + (float)a.S;
        for (int i = 0;; ++i) {
            const int s = i % CK_D, bi = i % CK_NB;
            mbar_wait(&sh.dfull[s], (i / CK_D) & 1);
            const RowDesc dsc = sh.dq[s];
            if (dsc.b < 0) break;
            mbar_wait(&sh.maxbar[s], (i / CK_D) & 1);  // the 8 slice maxima of row i
            if (lane == 0) TRACE(TR_MASS0, i, warp, 0);
#ifdef BS_TRACE
            const long long mc0 = clock64();
#endif
            float m = -INFINITY;
            uint32_t bad = 0;
            int g = 0x7FFFFFFF;
#pragma unroll
            for (int r = 0; r < CK_CL; ++r) {
                const uint4 cm = sh.cmax[s][r];
                m = fmaxf(m, __uint_as_float(cm.x));
                bad |= cm.y;
            }
#pragma unroll
            for (int r = 0; r < CK_CL; ++r)
                if (__uint_as_float(sh.cmax[s][r].x) == m) g = min(g, (int)sh.cmax[s][r].z);
            const bool ok = !bad && m > -INFINITY && fabsf(__fmul_rn(m, a.c)) < 16777216.0f;
            mbar_wait(&sh.full[bi], (i / CK_NB) & 1);  // (complete: the max warps read it)
            const uint16_t* buf = bufs + (size_t)bi * SL;
            uint64_t wacc = 0;
            if (a.T > 0.f && ok) {
                mp.nmc = -__fmul_rn(m, a.c);
                const int nfull = len / CK_TILE;  // whole tiles; the slice's ragged end follows
                auto tile_done = [&](int t, uint64_t acc) {
#ifdef BS_EXP_NOREDUX
                    wacc += acc;
#else
                    const uint64_t ts = warp_sum_u51(acc);
                    if (lane == 0) sh.tsum[s][t] = ts;
                    wacc += ts;
#endif
                };
                const uint32_t L02 = row_clamp_l0(mp.c, mp.nmc, a.S);
                if (L02) {  // the fast mass loop (bf16 pre-clamp, ALU unpack, F2I conversion)
                    // lane l: elements 8l.. and 256+8l.. of tile t (conflict-free 16-byte loads;
                    // the tile sum does not depend on which lane holds which element)
                    for (int t = warp; t < nfull; t += CK_NMW) {
                        const int e0 = t * CK_TILE + lane * 8;
                        tile_done(t, mass16_fast(lds128(buf + e0), lds128(buf + e0 + CK_TILE / 2), mp.c, mp.nmc,
                                                 mp.magic, L02));
                    }
                } else {
                    for (int t = warp; t < nfull; t += CK_NMW) {
                        const int e0 = t * CK_TILE + lane * 8;
                        tile_done(t, mass8(lds128(buf + e0), mp) + mass8(lds128(buf + e0 + CK_TILE / 2), mp));
                    }
                }
                if (nfull < ntile && warp == nfull % CK_NMW) {  // the ragged last tile
                    const int e0 = nfull * CK_TILE + lane * 16;
                    uint64_t acc = 0;
                    for (int x = 0; x < 16; ++x)
                        if (e0 + x < len) acc += mass_of(__uint_as_float((uint32_t)buf[e0 + x] << 16), mp);
                    tile_done(nfull, acc);
                }
            }
            if (lane == 0) sh.wsum[warp] = wacc;
#ifdef BS_TRACE
            if (lane == 0) TRACE(TR_MASSL, i, warp, (int)min(255ll, (clock64() - mc0) >> 6));
#endif
            named_bar(1, CK_NMW * 32);
            if (warp == 0) {
                uint64_t cs = 0;
#pragma unroll
                for (int w = 0; w < CK_NMW; ++w) cs += sh.wsum[w];
                const int dl = dsc.d - e_lo;
                const uint64_t mdl = (a.T > 0.f && ok && dsc.d >= 0 && dl >= 0 && dl < len)
                                         ? mass_of(__uint_as_float((uint32_t)buf[dl] << 16), mp)
                                         : 0ull;
                if (lane == 0) {
                    sh.erec[s] = make_uint4(__float_as_uint(m), bad, (uint32_t)g, 0u);
                    // arm row i's sum slot (its row i-4 phase completed: the max warps' eempty
                    // wait precedes this row's max); the arrive also releases the tile sums
                    // and erec to this CTA's epilogue
                    mbar_arrive_expect_tx(&sh.sumbar[s], (uint32_t)(CK_CL * 16));
                }
                __syncwarp();
                if (lane < CK_CL)
                    st_async_v4(&sh.csum[s][rank],
                                make_uint4((uint32_t)cs, (uint32_t)(cs >> 32), (uint32_t)mdl, (uint32_t)(mdl >> 32)),
                                &sh.sumbar[s], (uint32_t)lane);
            }
            named_bar(1, CK_NMW * 32);  // wsum reusable
            if (warp == 0 && lane == 0) TRACE(TR_MASS1, i, 0, 0);
            if (lane == 0) mbar_arrive(&sh.empty[bi]);  // slice buffer free
        }
    }
    cluster.sync();  // no CTA exits while a peer may still address its shared memory
    if (tid == 0) TRACE(TR_END, 0, 0, 0);
    if (tid == 0) {
        if (a.stats)
            for (int i = 0; i < STAT_COUNT; ++i)
                if (sh.stat[i]) atomicAdd(a.stats + i, sh.stat[i]);
    }
    // the last cluster out resets the scheduler words for the next launch (one exit atomic per
    // cluster: the cluster barrier above means its 8 CTAs are past every scheduler access)
    if (tid == 0 && rank == 0) {
        __threadfence();
        if (atomicAdd(a.sctl + SC_EXIT, 1u) == gridDim.x / CK_CL - 1) {
            a.sctl[SC_STATIC] = 0u;
            a.sctl[SC_NLIVE] = 0u;
            a.sctl[SC_PLANNED] = 0u;
            a.sctl[SC_DONE] = 0u;
            a.sctl[SC_EXIT] = 0u;
            a.sctl[SC_EPOCH] = (epoch + 1u) ? epoch + 1u : 1u;  // never 0 (zeroed entries)
            __threadfence();
        }
    }
}
