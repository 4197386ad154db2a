// lookup.cuh — the draft lookup of one rollout by one warp (K1: longest anchored
// suffix of the rollout's context in its prompt's pool, then the greedy continuation).
// Used by lookup_kernel (index.cu) and by the fused verify + commit + lookup launch
// (verify_cluster.cuh), which calls it with the just-committed state in registers.
#pragma once
#include "common.cuh"
#include "ctx.h"

namespace bs {

struct LookupArgs {
    const int32_t* slots;
    int n, k, M, Lmin;
    const int32_t* tail;
    const int32_t* ctx_len;
    const int32_t* prompt;
    const int32_t* pos;
    const int32_t* max_len;
    const int32_t* finished;
    const IndexDesc* desc;  // the sealed index (device-resident: stable across RL steps)
    const unsigned long long* cur_step;  // rl_step of the latest put / seal (staleness)
    uint32_t* dev_err;
    int32_t* draft;
    int32_t* draft_len;
    int32_t* match_len;
};

__device__ __forceinline__ bool probe(const IndexEntry* table, uint64_t mask, uint64_t key,
                                      uint32_t& occ, uint32_t& meta) {
    uint64_t s = key & mask;
    for (;;) {
        const uint4 e = __ldg(reinterpret_cast<const uint4*>(table + s));
        const uint64_t k = ((uint64_t)e.y << 32) | e.x;
        if (k == key) {
            occ = e.z;
            meta = e.w;
            return true;
        }
        if (k == 0) return false;
        s = (s + 1) & mask;
    }
}

// HASH_B^i for the lookup's per-lane suffix hash (a warp scan of y[-1-i] * B^i).
struct HashPow {
    uint64_t v[32];
};
constexpr HashPow make_hash_pow() {
    HashPow t{};
    uint64_t x = 1;
    for (int i = 0; i < 32; ++i) {
        t.v[i] = x;
        x *= HASH_B;
    }
    return t;
}
__constant__ HashPow c_hash_pow = make_hash_pow();

// Rollout b's draft for its next step from its state: context length L, prompt P, position p,
// max length ml, finished flag fin, and lane i's context token y[-1-i] (tok_raw, lane < M).
// Writes draft[b, 0..k), draft_len[b], match_len[b].  Whole warp.
// stale: the index was sealed for another rl_step than the latest put (a hard
// error): the draft is empty and the error word says so.
__device__ __forceinline__ void lookup_rollout(const LookupArgs& a, const IndexDesc& x, int b, int L, int P, int p,
                                               int ml, bool fin, int tok_raw, int lane, bool stale) {
    const int M = a.M;
    if (stale && lane == 0) atomicOr(a.dev_err, DEV_STALE);
    fin = fin || p >= ml || stale;
    const int mmax = min(M, L);
    const int tok = (lane < mmax) ? tok_raw : -1;
    uint64_t H = (lane < mmax) ? (uint64_t)(uint32_t)(tok + 1) * c_hash_pow.v[lane] : 0ull;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
        const uint32_t lo = __shfl_up_sync(0xFFFFFFFFu, (uint32_t)H, dd);
        const uint32_t hi = __shfl_up_sync(0xFFFFFFFFu, (uint32_t)(H >> 32), dd);
        if (lane >= dd) H += ((uint64_t)hi << 32) | lo;
    }
    uint32_t occ = 0, meta = 0;
    bool found = false;
    if (!fin && lane < mmax) found = probe(x.table, x.mask, window_key(H, P, lane + 1), occ, meta);
    unsigned hit = __ballot_sync(0xFFFFFFFFu, found);
    int mstar = 0, q = 0, dstart = 0;
    int dpre = -1;        // T[dstart + lane], prefetched when the draft is the m0 window's
    bool dpre_ok = false;
    for (;;) {
        if (hit == 0) break;
        const int m0 = 32 - __clz(hit);  // largest stored suffix length
        const uint32_t occ0 = __shfl_sync(0xFFFFFFFFu, occ, m0 - 1);
        const uint32_t meta0 = __shfl_sync(0xFFFFFFFFu, meta, m0 - 1);
        const bool uniq = (meta0 & META_UNIQUE) && (meta0 & META_CONT);
        // one round trip: the anchor check y[-m0:] == T[occ0 .. occ0+m0) (guards a 64-bit
        // key false positive), the continuation T[occ0+m0 ..] (the draft if this anchor wins;
        // meta's q tokens exist) and, for a unique window, its left extension T[occ0-1-lane]
        // and its sequence start
        const int qm = (int)(meta0 & 0xFFu);
        const int tchk = (lane < m0) ? x.T[(int64_t)occ0 + m0 - 1 - lane] : 0;
        const int tcont = (lane < qm) ? x.T[(int64_t)occ0 + m0 + lane] : -1;
        const int text = (uniq && (int64_t)occ0 - 1 - lane >= 0) ? x.T[(int64_t)occ0 - 1 - lane] : -2;
        const int sstart = uniq ? x.seq_start_of[occ0] : 0;
        const bool okc = (lane >= m0) || (tchk == tok);
        if (!__all_sync(0xFFFFFFFFu, okc)) {
            hit &= ~(1u << (m0 - 1));
            continue;
        }
        if (uniq) {
            // unique occurrence: extend the anchor to the left within its sequence
            const int jj = lane;  // compare y[-m0-1-jj] with T[occ0-1-jj]
            const int yt = __shfl_sync(0xFFFFFFFFu, tok_raw, (m0 + jj) & 31);
            bool eq = false;
            if (m0 + jj < mmax && (int64_t)occ0 - 1 - jj >= sstart) eq = (text == yt);
            const unsigned eqm = __ballot_sync(0xFFFFFFFFu, eq);
            const int ext = (~eqm == 0u) ? 32 : (__ffs(~eqm) - 1);
            mstar = m0 + ext;
            q = qm;
            dstart = (int)occ0 + m0;
            dpre = tcont;
            dpre_ok = true;
            break;
        }
        // longest stored suffix with a continuation (non-unique entries, <= m0)
        const unsigned lim = (meta0 & META_UNIQUE) ? ((1u << (m0 - 1)) - 1u)
                                                   : (m0 == 32 ? 0xFFFFFFFFu : ((1u << m0) - 1u));
        const unsigned contm = __ballot_sync(0xFFFFFFFFu, found && (meta & META_CONT)) & hit & lim;
        if (contm == 0) break;
        const int ms = 32 - __clz(contm);
        if (ms == m0) {  // the checked m0 window itself: its continuation is already loaded
            mstar = m0;
            q = qm;
            dstart = (int)occ0 + m0;
            dpre = tcont;
            dpre_ok = true;
            break;
        }
        const uint32_t occs = __shfl_sync(0xFFFFFFFFu, occ, ms - 1);
        const uint32_t metas = __shfl_sync(0xFFFFFFFFu, meta, ms - 1);
        bool oks = true;
        if (lane < ms) oks = (x.T[(int64_t)occs + ms - 1 - lane] == tok);
        if (!__all_sync(0xFFFFFFFFu, oks)) {
            hit &= ~(1u << (ms - 1));
            continue;
        }
        mstar = ms;
        q = (int)(metas & 0xFFu);
        dstart = (int)occs + ms;
        break;
    }
    if (mstar < a.Lmin) {
        mstar = 0;
        q = 0;
    }
    if (fin) {
        mstar = 0;
        q = 0;
    }
    q = min(q, a.k);
    q = min(q, max(0, ml - p - 1));
    if (lane < a.k) a.draft[(int64_t)b * a.k + lane] = (lane < q) ? (dpre_ok ? dpre : x.T[(int64_t)dstart + lane]) : -1;
    if (lane == 0) {
        a.draft_len[b] = q;
        if (a.match_len) a.match_len[b] = mstar;
    }
}

}  // namespace bs
