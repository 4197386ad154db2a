// verify.cu — fused vocab-row verify + resample (Eq. 2, Eq. 3 P:208-210,
// Alg. 1, bonus token P:308) for sm_100a.
//
// Kernel K3.  A PERSISTENT grid of thread-block clusters; a cluster of C
// CTAs owns one logits row at a time, CTA `rank` the vocabulary slice
// [rank*SL, (rank+1)*SL).  Work is claimed per ROLLOUT (one atomic each) and a rollout's
// rows are verified in Alg. 1's order, lazily: row j+1 is read only if row j accepted
// d_{j+1} (rows after the first rejection are never read).
//
// Each cluster keeps two rollouts in flight ("slots" A and B) and runs the three stages
// of a row — P1 (row max), P2 (integer masses, exact sums), DEC (accept / sample) — on
// the fixed software-pipelined schedule  P1(A) DEC(B) P2(A) P1(B) DEC(A) P2(B), so the
// TMA load of a slot's next row streams in under the other slot's mass pass.  The
// cross-CTA reductions are point-to-point: every CTA pushes its slice record into all
// peers' shared memory (DSMEM stores) and arrives remotely on their mbarrier
// (release.cluster); one thread per consumer CTA waits (acquire.cluster) and a CTA
// barrier orders the rest — there is no cluster-wide barrier in the loop.  All
// control-path global loads (row numbers, draft tokens, the next rollout) are issued by
// thread 0 one stage early and published through shared memory.
//   * P1: NaN-propagating bf16x2 max over the slice (1-D bulk async copies on the TMA
//     engine, mbarrier completion, L2 evict-first);
//   * P2: masses of reading R with packed FFMA2/FADD2, exact u64 per-warp sums;
//   * DEC: Z, mass(d) -> accept (Philox counter (pos+j, ACCEPT), drawn under P1); a
//     residual / bonus sample is found by the CTA holding the CDF crossing: all its
//     warps sum the crossing warp's tiles in parallel, one warp scans the crossing tile.
#include <cooperative_groups.h>
#include <cstdlib>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "ctx.h"
#include "ptx.cuh"

namespace cg = cooperative_groups;

namespace bs {

constexpr int MAXC = 16;  // max cluster size (16 is non-portable; B200 supports it)

// Optional per-stage cycle accounting (build with -DBS_PHASE_TIMING; read with
// bsx_phase_times): thread 0 of every CTA adds the clock64() delta of each stage.
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

struct VerifyArgs {
    const int32_t* slots;
    const uint16_t* logits;
    const int64_t* row_index;
    int64_t stride;
    const int32_t* draft;
    int32_t k, V, SL, C, ntiles, S, eos;
    float T, c;
    unsigned long long seed;
    const int32_t* pos;
    const unsigned long long* uid;
    const int32_t* rb_q;
    const int32_t* active;  // compacted live rollouts (plan kernel)
    unsigned int* ctl;      // VCTL_* words
    uint32_t* dev_err;
    int32_t* out_tokens;
    int32_t* out_len;
    int32_t* out_acc;
    float* out_norm;
    unsigned long long* out_z;
    unsigned long long* stats;
};

// Records pushed to every CTA of the cluster (index = source rank), double-buffered by
// row parity so a producer one row ahead never overwrites an unread record.
struct MaxRec {
    float max;
    uint32_t bad;
    int32_t spare;  // rank 0 only: the slot's claimed-ahead next rollout (-1: none left)
    int32_t pad;
};
struct SumRec {
    unsigned long long sum;    // slice mass sum (greedy: first argmax index)
    unsigned long long massd;  // mass of the draft token if it lies in the slice
};

// Slot metadata, written by thread 0 (issuer), read by every thread after a barrier.
struct SlotMeta {
    int32_t b, j, q, d;  // rollout, row, clamped draft length, d_{j+1} (-1 if j == q)
    int32_t bulk;        // elements of this CTA's slice staged by the bulk copy
    int32_t pad[3];
};

struct __align__(16) VShared {
    uint64_t full[2];     // TMA completion, one per slot buffer
    uint64_t bar_max[2];  // C arrivals per row: slice maxima of the slot's row
    uint64_t bar_sum[2];  // C arrivals per row: slice sums of the slot's row
    MaxRec rmax[2][2][MAXC];
    SumRec rsum[2][2][MAXC];
    SlotMeta meta[2];
    int32_t init_rollouts[4];
    // CTA-local
    float wmax[32];
    uint32_t wbad[32];
    unsigned long long wsum[2][32];  // per slot: exact per-warp sums (sample search)
    unsigned long long tsum[32];     // sample search: sums of the crossing warp's tiles
    uint32_t rng[2][8];              // per slot: Philox ACCEPT (0-3) and SAMPLE (4-7) draws
    unsigned long long stat[STAT_COUNT];
};

// ------------------------------------------------------------------ packed fp32 math
struct F2 {
    float x, y;
};
__device__ __forceinline__ F2 ffma2(F2 a, F2 b, F2 c) {
    F2 r;
    asm("{\n .reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " mov.b64 rc, {%6, %7};\n fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return r;
}
__device__ __forceinline__ F2 fadd2(F2 a, F2 b) {
    F2 r;
    asm("{\n .reg .b64 ra, rb, rd;\n mov.b64 ra, {%2, %3};\n mov.b64 rb, {%4, %5};\n"
        " add.rn.f32x2 rd, ra, rb;\n mov.b64 {%0, %1}, rd;\n}"
        : "=f"(r.x), "=f"(r.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return r;
}

// Masses of the two bf16 logits packed in w (R2-R4), bit-identical to mass_of() per lane:
// the packed FFMA2 / FADD2 perform the same IEEE single operations.
__device__ __forceinline__ void mass_pair(uint32_t w, const MassParams& mp, uint64_t& m0,
                                          uint64_t& m1) {
    const F2 l{bf16lo(w), bf16hi(w)};
    F2 y = ffma2(l, F2{mp.c, mp.c}, F2{mp.nmc, mp.nmc});
    y.x = fmaxf(y.x, mp.clampv);
    y.y = fmaxf(y.y, mp.clampv);
    const F2 t = fadd2(y, F2{mp.magic, mp.magic});
    const F2 n = fadd2(t, F2{-mp.magic, -mp.magic});
    const F2 f = fadd2(y, F2{-n.x, -n.y});
    F2 p = ffma2(F2{BS_C5, BS_C5}, f, F2{BS_C4, BS_C4});
    p = ffma2(p, f, F2{BS_C3, BS_C3});
    p = ffma2(p, f, F2{BS_C2, BS_C2});
    p = ffma2(p, f, F2{BS_C1, BS_C1});
    p = ffma2(p, f, F2{BS_C0, BS_C0});
    m0 = f2u64_rz(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)));
    m1 = f2u64_rz(__uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

__device__ __forceinline__ uint64_t mass8(const uint4 v, const MassParams& mp) {
    uint64_t a0, a1, b0, b1, c0, c1, d0, d1;
    mass_pair(v.x, mp, a0, a1);
    mass_pair(v.y, mp, b0, b1);
    mass_pair(v.z, mp, c0, c1);
    mass_pair(v.w, mp, d0, d1);
    return ((a0 + a1) + (b0 + b1)) + ((c0 + c1) + (d0 + d1));
}

// Masses of one lane's 8 elements of a tile with element `excl` (slice-local) zeroed.
__device__ __forceinline__ void mass8_excl(const uint4 v, const MassParams& mp, int e0, int excl,
                                           uint64_t mm[8]) {
    mass_pair(v.x, mp, mm[0], mm[1]);
    mass_pair(v.y, mp, mm[2], mm[3]);
    mass_pair(v.z, mp, mm[4], mm[5]);
    mass_pair(v.w, mp, mm[6], mm[7]);
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (e0 + i == excl) mm[i] = 0;
}

__device__ __forceinline__ uint32_t hmax2_nan_u32(uint32_t a, uint32_t b) {
    __nv_bfloat162 x, y;
    memcpy(&x, &a, 4);
    memcpy(&y, &b, 4);
    __nv_bfloat162 z = __hmax2_nan(x, y);
    uint32_t r;
    memcpy(&r, &z, 4);
    return r;
}

__device__ __forceinline__ float bf16_at(const uint16_t* sl, int e) {
    return __uint_as_float((uint32_t)sl[e] << 16);
}

// ------------------------------------------------------------------ helpers per row
__device__ __forceinline__ int64_t row_no(const VerifyArgs& a, int b, int j) {
    const int kp1 = a.k + 1;
    return a.row_index ? a.row_index[(int64_t)b * kp1 + j] : (int64_t)b * kp1 + j;
}

// Issue the bulk copy of this CTA's slice of logits row `rowno` into `buf` (thread 0);
// returns the number of elements the bulk copy stages (the rest is loaded by the CTA).
__device__ __forceinline__ int issue_load(const VerifyArgs& a, int64_t rowno, int rank,
                                          uint16_t* buf, uint64_t* bar, uint64_t pol) {
    const int s0 = rank * a.SL, s1 = min(a.V, s0 + a.SL);
    const int len = max(0, s1 - s0);
    const uint16_t* src = a.logits + rowno * a.stride + s0;
    const bool aligned = ((reinterpret_cast<uintptr_t>(src) & 15u) == 0);
    const int bulk = aligned ? (len & ~7) : 0;
    fence_proxy_async_smem();
    if (bulk) {
        mbar_arrive_expect_tx(bar, (uint32_t)bulk * 2u);
        constexpr int CH = 8192;  // elements per bulk copy (16 KiB)
        for (int off = 0; off < bulk; off += CH)
            bulk_g2s(buf + off, src + off, (uint32_t)min(CH, bulk - off) * 2u, bar, pol);
    } else {
        mbar_arrive(bar);
    }
    return bulk;
}

// Alg. 1 lines 10-31 for rollout b decided at row j (all rows < j accepted).
__device__ void finalize_rollout(const VerifyArgs& a, VShared& sh, int b, int j, int q,
                                 bool accept_eos, int cand) {
    const int kp1 = a.k + 1;
    int32_t* out = a.out_tokens + (int64_t)b * kp1;
    const int32_t* d = a.draft + (int64_t)b * a.k;
    int n = 0;
    for (int i = 0; i < j; ++i) out[n++] = d[i];
    int acc = j;
    if (accept_eos) {
        out[n++] = d[j];
        acc = j + 1;
    } else {
        out[n++] = cand;
    }
    for (int i = n; i < kp1; ++i) out[i] = -1;
    a.out_len[b] = n;
    a.out_acc[b] = acc;
    if (a.stats) {  // CTA-local counters, flushed once at kernel exit
        unsigned long long* st = sh.stat;
        if (q > 0) {
            atomicAdd(st + STAT_STEPS_SPEC, 1ull);
            atomicAdd(st + STAT_EMIT_SPEC, (unsigned long long)n);
            atomicAdd(st + STAT_ACCEPTED, (unsigned long long)acc);
            atomicAdd(st + STAT_PROPOSED, (unsigned long long)q);
            atomicAdd(st + STAT_HIST + min(n, STAT_HIST_BINS - 1), 1ull);
        } else {
            atomicAdd(st + STAT_STEPS_PLAIN, 1ull);
            atomicAdd(st + STAT_EMIT_PLAIN, (unsigned long long)n);
        }
        atomicAdd(st + STAT_ROWS_VERIFIED, (unsigned long long)(j + 1));
        atomicAdd(st + STAT_ROWS_NEEDED, (unsigned long long)(j + 1));
    }
}

enum { ST_P1 = 0, ST_P2 = 1, ST_DEC = 2, ST_EMPTY = 3 };

// Thread 0's prefetched successors of a slot (registers of thread 0 only).
struct Prefetch {
    int64_t next_row;  // row (b, j+1)
    int next_d;        // d_{j+2} (-1 when j+1 == q)
    int nb, nq, nd;    // the spare rollout: b, q, d_1
    int64_t nrow0;     // its row 0
};

template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) verify_rows_kernel(const VerifyArgs a) {
    constexpr int NW = NT / 32;
    cg::cluster_group cluster = cg::this_cluster();
    const int C = a.C;
    const int rank = (int)cluster.block_rank();
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint16_t* bufs[2] = {reinterpret_cast<uint16_t*>(smem_raw),
                         reinterpret_cast<uint16_t*>(smem_raw) + (size_t)a.ntiles * 256};
    VShared& sh = *reinterpret_cast<VShared*>(smem_raw + (size_t)a.ntiles * 1024);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int kp1 = a.k + 1;
    const int s0 = rank * a.SL;
    const int s1 = min(a.V, s0 + a.SL);
    const int len = max(0, s1 - s0);
    const int ntl = (len + 255) >> 8;        // 256-element tiles in this slice
    const int tpw = (ntl + NW - 1) / NW;     // tiles per warp (contiguous ranges)
    const int t0 = min(ntl, warp * tpw), t1 = min(ntl, t0 + tpw);
    const uint64_t pol = policy_evict_first();
    const int nact = (int)a.ctl[VCTL_NACTIVE];
    MassParams mp;
    mp.c = a.c;
    mp.clampv = -(float)(a.S + 2);
    mp.magic = 12582912.0f + (float)a.S;

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sh.full[i], 1);
            mbar_init(&sh.bar_max[i], 1);  // one local arrive.expect_tx + C*16 async bytes
            mbar_init(&sh.bar_sum[i], 1);
        }
        fence_mbar_init();
        for (int i = 0; i < 2; ++i) {  // arm the first phase of every exchange barrier
            mbar_arrive_expect_tx(&sh.bar_max[i], (uint32_t)C * 16u);
            mbar_arrive_expect_tx(&sh.bar_sum[i], (uint32_t)C * 16u);
        }
    }
    for (int i = tid; i < STAT_COUNT; i += NT) sh.stat[i] = 0ull;
    for (int e = len + tid; e < a.ntiles * 256; e += NT) {  // -inf padding past the slice
        bufs[0][e] = (uint16_t)0xFF80u;
        bufs[1][e] = (uint16_t)0xFF80u;
    }
    // leader claims two rollouts + one spare per slot
    int spare_reg[2] = {-1, -1};  // meaningful in the leader thread only
    if (rank == 0 && tid == 0) {
        const int base = (int)atomicAdd(a.ctl + VCTL_NEXT, 4u);
        for (int rr = 0; rr < C; ++rr) {
            VShared* o = cluster.map_shared_rank(&sh, rr);
            o->init_rollouts[0] = base;
            o->init_rollouts[1] = base + 1;
        }
        spare_reg[0] = (base + 2 < nact) ? base + 2 : -1;
        spare_reg[1] = (base + 3 < nact) ? base + 3 : -1;
    }
    __syncthreads();
    cluster.sync();
    int stage[2], par[2];
    Prefetch pf[2];
    for (int x = 0; x < 2; ++x) {
        const int ri = sh.init_rollouts[x];
        stage[x] = (ri < nact) ? ST_P1 : ST_EMPTY;
        par[x] = 0;
        if (tid == 0 && ri < nact) {
            const int b = a.active[ri];
            const int q = a.rb_q[b];
            SlotMeta& mt = sh.meta[x];
            mt.b = b;
            mt.j = 0;
            mt.q = q;
            mt.d = (q > 0) ? a.draft[(int64_t)b * a.k] : -1;
            mt.bulk = issue_load(a, row_no(a, b, 0), rank, bufs[x], &sh.full[x], pol);
        }
    }
    __syncthreads();
    uint32_t fph[2] = {0u, 0u}, mph[2] = {0u, 0u}, sph[2] = {0u, 0u};  // barrier phases
    float mrow[2] = {0.f, 0.f};
    bool okrow[2] = {true, true};
#ifdef BS_PHASE_TIMING
    long long ph_t = clock64();
#endif

    // ------------------------------------------------------------ stage bodies
    auto stage_p1 = [&](int x) {
        uint16_t* sl = bufs[x];
        __syncthreads();  // meta[x] was rewritten by thread 0 when the slot advanced
        const SlotMeta mt = sh.meta[x];
        if (warp == NW - 1 && lane < 2) {  // the row's two Philox draws (one per lane), in
            const int slot = a.slots[mt.b];  // the warp with the fewest max/mass tiles
            const uint64_t uidv = a.uid[slot];
            const uint32_t position = (uint32_t)(a.pos[slot] + mt.j);
            const U128 r = draw(a.seed, uidv, position, lane ? PURPOSE_SAMPLE : PURPOSE_ACCEPT);
            uint32_t* o = sh.rng[x] + 4 * lane;
            o[0] = r.x0; o[1] = r.x1; o[2] = r.x2; o[3] = r.x3;
        }
        mbar_wait(&sh.full[x], fph[x]);
        fph[x] ^= 1u;
        PH_MARK(1);
        if (mt.bulk < len) {  // ragged part (unaligned rows / slice length not a multiple of 8)
            const uint16_t* src = a.logits + row_no(a, mt.b, mt.j) * a.stride + s0;
            for (int e = mt.bulk + tid; e < len; e += NT) sl[e] = src[e];
            __syncthreads();
        }
        uint32_t mx = 0xFF80FF80u;
        for (int t = t0; t < t1; ++t) {
            const uint4 v = lds128(sl + t * 256 + lane * 8);
            mx = hmax2_nan_u32(mx, v.x);
            mx = hmax2_nan_u32(mx, v.y);
            mx = hmax2_nan_u32(mx, v.z);
            mx = hmax2_nan_u32(mx, v.w);
        }
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
        __syncthreads();
        const int spv = __shfl_sync(0xFFFFFFFFu, spare_reg[x], 0);  // the leader's, in warp 0
        if (tid < C) {  // push this slice's record into CTA `tid`, then arrive there
            MaxRec r;
            r.max = -INFINITY;
            r.bad = 0;
            for (int w = 0; w < NW; ++w) {
                r.max = fmaxf(r.max, sh.wmax[w]);
                r.bad |= sh.wbad[w];
            }
            r.spare = (rank == 0) ? spv : -1;
            r.pad = 0;
            uint4 v;
            memcpy(&v, &r, 16);
            st_async_v4(&sh.rmax[x][par[x]][rank], v, &sh.bar_max[x], (uint32_t)tid);
        }
        stage[x] = ST_P2;
        PH_MARK(2);
    };

    auto stage_p2 = [&](int x) {
        uint16_t* sl = bufs[x];
        // the peers' records landed with their transaction bytes (st.async): a CTA-scope
        // wait suffices; thread 0 then arms the barrier for the slot's next row
        mbar_wait(&sh.bar_max[x], mph[x]);
        mph[x] ^= 1u;
        if (tid == 0) mbar_arrive_expect_tx(&sh.bar_max[x], (uint32_t)C * 16u);
        PH_MARK(3);
        const SlotMeta mt = sh.meta[x];
        const MaxRec* rec = sh.rmax[x][par[x]];
        if (tid == 0) {  // prefetch the slot's successors (consumed at DEC)
            Prefetch& p = pf[x];
            if (mt.j < mt.q) {
                p.next_row = row_no(a, mt.b, mt.j + 1);
                p.next_d = (mt.j + 1 < mt.q) ? a.draft[(int64_t)mt.b * a.k + mt.j + 1] : -1;
            }
            const int nri = rec[0].spare;
            if (nri >= 0) {
                p.nb = a.active[nri];
                p.nq = a.rb_q[p.nb];
                p.nd = (p.nq > 0) ? a.draft[(int64_t)p.nb * a.k] : -1;
                p.nrow0 = row_no(a, p.nb, 0);
            }
        }
        float m = -INFINITY;
        uint32_t bb = 0;
        for (int rr = 0; rr < C; ++rr) {
            m = fmaxf(m, rec[rr].max);
            bb |= rec[rr].bad;
        }
        bool ok = true;
        uint32_t err = 0;
        if (bb) { ok = false; err |= DEV_BAD_LOGIT; }
        else if (m == -INFINITY) { ok = false; err |= DEV_ALL_NEGINF; }
        else if (a.T > 0.f && !(fabsf(__fmul_rn(m, a.c)) < 16777216.0f)) { ok = false; err |= DEV_RANGE; }
        if (err && rank == 0 && tid == 0) atomicOr(a.dev_err, err);
        mrow[x] = m;
        okrow[x] = ok;
        SumRec out;
        out.massd = 0ull;
        if (a.T == 0.f) {  // greedy (R1): first index attaining the max
            int first = 0x7FFFFFFF;
            if (ok) {
                for (int t = t0; t < t1 && first == 0x7FFFFFFF; ++t) {
                    const int e0 = t * 256 + lane * 8;
                    const uint4 v = lds128(sl + e0);
                    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
                    int f = 0x7FFFFFFF;
#pragma unroll
                    for (int i = 3; i >= 0; --i) {
                        if (bf16hi(w4[i]) == m) f = e0 + 2 * i + 1;
                        if (bf16lo(w4[i]) == m) f = e0 + 2 * i;
                    }
#pragma unroll
                    for (int mm = 16; mm; mm >>= 1) f = min(f, __shfl_xor_sync(0xFFFFFFFFu, f, mm));
                    first = f;
                }
            }
            if (lane == 0) sh.wsum[x][warp] = (unsigned long long)(uint32_t)first;
            __syncthreads();
            int f = 0x7FFFFFFF;
            for (int w = 0; w < NW; ++w) f = min(f, (int)sh.wsum[x][w]);
            out.sum = (unsigned long long)(uint32_t)((f == 0x7FFFFFFF) ? f : s0 + f);
        } else {  // integer masses (R2-R4), exact sums
            mp.nmc = -__fmul_rn(m, a.c);
            uint64_t acc0 = 0, acc1 = 0;
            if (ok) {
                int t = t0;
                for (; t + 1 < t1; t += 2) {  // two tiles per step: 8 independent pair chains
                    const uint4 v0 = lds128(sl + t * 256 + lane * 8);
                    const uint4 v1 = lds128(sl + (t + 1) * 256 + lane * 8);
                    acc0 += mass8(v0, mp);
                    acc1 += mass8(v1, mp);
                }
                if (t < t1) acc0 += mass8(lds128(sl + t * 256 + lane * 8), mp);
            }
            const uint64_t acc = warp_sum_u64(acc0 + acc1);
            if (lane == 0) sh.wsum[x][warp] = acc;
            __syncthreads();
            uint64_t sum = 0;
            for (int w = 0; w < NW; ++w) sum += sh.wsum[x][w];
            out.sum = sum;
            if (ok && mt.d >= s0 && mt.d < s1) out.massd = mass_of(bf16_at(sl, mt.d - s0), mp);
        }
        if (tid < C) {
            uint4 v;
            memcpy(&v, &out, 16);
            st_async_v4(&sh.rsum[x][par[x]][rank], v, &sh.bar_sum[x], (uint32_t)tid);
        }
        stage[x] = ST_DEC;
        PH_MARK(4);
    };

    auto stage_dec = [&](int x) {
        uint16_t* sl = bufs[x];
        mbar_wait(&sh.bar_sum[x], sph[x]);
        sph[x] ^= 1u;
        if (tid == 0) mbar_arrive_expect_tx(&sh.bar_sum[x], (uint32_t)C * 16u);
        PH_MARK(5);
        const SlotMeta mt = sh.meta[x];
        const int j = mt.j, q = mt.q, d = mt.d, b = mt.b;
        const bool ok = okrow[x];
        const SumRec* rs = sh.rsum[x][par[x]];
        bool finished;
        if (a.T == 0.f) {
            int g = 0x7FFFFFFF;
            for (int rr = 0; rr < C; ++rr) g = min(g, (int)(uint32_t)rs[rr].sum);
            g = ok ? g : -1;
            const bool accepted = ok && j < q && d == g;
            const bool eos_acc = accepted && a.eos >= 0 && d == a.eos;
            finished = !accepted || eos_acc;
            if (rank == 0 && tid == 0) {
                if (a.out_norm) a.out_norm[(int64_t)b * kp1 + j] = ok ? 1.0f : 0.f;
                if (a.out_z) a.out_z[(int64_t)b * kp1 + j] = ok ? 1ull : 0ull;
                if (finished) finalize_rollout(a, sh, b, j, q, eos_acc, g);
            }
        } else {
            uint64_t Zs = 0, md = 0;
            for (int rr = 0; rr < C; ++rr) {
                Zs += rs[rr].sum;
                md += rs[rr].massd;
            }
            bool accepted = false;
            if (ok && j < q) {
                const U128 r1{sh.rng[x][0], sh.rng[x][1], sh.rng[x][2], sh.rng[x][3]};
                accepted = uniform_floor(r1, Zs) < md;
            }
            const bool eos_acc = accepted && a.eos >= 0 && d == a.eos;
            finished = !accepted || eos_acc;
            if (rank == 0 && tid == 0) {
                const uint64_t Zo = ok ? Zs : 0ull;
                if (a.out_norm) a.out_norm[(int64_t)b * kp1 + j] = ok ? (float)ldexp((double)Zo, -a.S) : 0.f;
                if (a.out_z) a.out_z[(int64_t)b * kp1 + j] = Zo;
                if (!ok) finalize_rollout(a, sh, b, j, q, false, -1);
                else if (eos_acc) finalize_rollout(a, sh, b, j, q, true, -1);
            }
            if (ok && finished && !eos_acc) {
                // residual (rejection: d excluded) or bonus sample (R8): which CTA holds the
                // CDF crossing?  (computed redundantly, no synchronisation)
                const int excl = (j < q) ? d : -1;
                const U128 r2{sh.rng[x][4], sh.rng[x][5], sh.rng[x][6], sh.rng[x][7]};
                const uint64_t U2 = uniform_floor(r2, Zs - ((j < q) ? md : 0ull));
                uint64_t before = 0;
                int cross = -1;
                uint64_t ul = 0;
                for (int rr = 0; rr < C; ++rr) {
                    const int r0 = rr * a.SL, r1e = min(a.V, r0 + a.SL);
                    const uint64_t adj = rs[rr].sum - ((excl >= r0 && excl < r1e) ? md : 0ull);
                    if (U2 < before + adj) {
                        cross = rr;
                        ul = U2 - before;
                        break;
                    }
                    before += adj;
                }
                if (cross == rank) {  // this CTA samples (uniform inside the CTA)
                    const int lex = excl - s0;  // slice-local excluded index
                    int wstar = 0;
                    before = 0;
                    for (int w = 0; w < NW; ++w) {
                        const int w0 = w * tpw * 256, w1 = min(len, w0 + tpw * 256);
                        const uint64_t adj = sh.wsum[x][w] - ((lex >= w0 && lex < w1) ? md : 0ull);
                        if (ul < before + adj) {
                            wstar = w;
                            ul -= before;
                            break;
                        }
                        before += adj;
                    }
                    mp.nmc = -__fmul_rn(mrow[x], a.c);
                    // tile sums of the crossing warp's tiles, all warps in parallel
                    const int c0 = min(ntl, wstar * tpw), c1 = min(ntl, c0 + tpw);
                    for (int t = c0 + warp; t < c1; t += NW) {
                        uint64_t mm[8];
                        mass8_excl(lds128(sl + t * 256 + lane * 8), mp, t * 256 + lane * 8, lex, mm);
                        uint64_t ls = 0;
#pragma unroll
                        for (int i = 0; i < 8; ++i) ls += mm[i];
                        ls = warp_sum_u64(ls);
                        if (lane == 0) sh.tsum[t - c0] = ls;
                    }
                    __syncthreads();
                    if (warp == 0) {  // crossing tile, then the crossing lane and element
                        int tstar = c0;
                        uint64_t ut = ul;
                        for (int t = c0; t < c1; ++t) {
                            const uint64_t ts = sh.tsum[t - c0];
                            if (ut < ts) {
                                tstar = t;
                                break;
                            }
                            ut -= ts;
                        }
                        uint64_t mm[8];
                        const int e0 = tstar * 256 + lane * 8;
                        mass8_excl(lds128(sl + e0), mp, e0, lex, mm);
                        uint64_t ls = 0;
#pragma unroll
                        for (int i = 0; i < 8; ++i) ls += mm[i];
                        const uint64_t incl = warp_incl_scan_u64(ls, lane);
                        const unsigned hit = __ballot_sync(0xFFFFFFFFu, ut < incl);
                        const int L = hit ? (__ffs(hit) - 1) : 31;
                        if (lane == L) {
                            uint64_t cum = incl - ls;
                            int tok = -1;
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                cum += mm[i];
                                if (tok < 0 && cum > ut) tok = s0 + e0 + i;
                            }
                            finalize_rollout(a, sh, b, j, q, false, tok);
                        }
                    }
                }
            }
        }
        PH_MARK(6);
        // ---- advance the slot: the next row of this rollout, or the slot's spare rollout
        const int nri = sh.rmax[x][par[x]][0].spare;  // broadcast with this row's P1
        par[x] ^= 1;
        if (!finished) {
            stage[x] = ST_P1;
            if (tid == 0) {
                SlotMeta& m2 = sh.meta[x];
                m2.j = j + 1;
                m2.d = pf[x].next_d;
                m2.bulk = issue_load(a, pf[x].next_row, rank, bufs[x], &sh.full[x], pol);
            }
        } else {
            __syncthreads();  // the sampling warps are done with bufs[x] and meta[x]
            if (nri >= 0) {
                stage[x] = ST_P1;
                if (tid == 0) {
                    SlotMeta& m2 = sh.meta[x];
                    m2.b = pf[x].nb;
                    m2.j = 0;
                    m2.q = pf[x].nq;
                    m2.d = pf[x].nd;
                    m2.bulk = issue_load(a, pf[x].nrow0, rank, bufs[x], &sh.full[x], pol);
                }
                if (rank == 0 && tid == 0) {  // claim the next spare for this slot
                    const int c2 = (int)atomicAdd(a.ctl + VCTL_NEXT, 1u);
                    spare_reg[x] = (c2 < nact) ? c2 : -1;
                }
            } else {
                stage[x] = ST_EMPTY;
            }
        }
        PH_MARK(7);
#ifdef BS_PHASE_TIMING
        if (tid == 0) atomicAdd(&g_phase[15], 1ull);
#endif
    };

    // ------------------------------------------------------------ the pipelined schedule
    for (;;) {
        PH_MARK(0);
        if (stage[0] == ST_P1) stage_p1(0);
        if (stage[1] == ST_DEC) stage_dec(1);
        if (stage[0] == ST_P2) stage_p2(0);
        if (stage[1] == ST_P1) stage_p1(1);
        if (stage[0] == ST_DEC) stage_dec(0);
        if (stage[1] == ST_P2) stage_p2(1);
        if (stage[0] == ST_EMPTY && stage[1] == ST_EMPTY) break;
    }
    // flush the CTA's statistics counters
    __syncthreads();
    if (a.stats)
        for (int i = tid; i < STAT_COUNT; i += NT)
            if (sh.stat[i]) atomicAdd(a.stats + i, sh.stat[i]);
    cluster.sync();  // no CTA exits while a peer may still access its shared memory
}

// ---- plan: clamp q per rollout, compact the live rollouts (one block)
constexpr int PLAN_NT = 1024;
__global__ void __launch_bounds__(PLAN_NT) verify_plan_kernel(
    int n, int k, int V, const int32_t* slots, const int32_t* draft, const int32_t* draft_len,
    const int32_t* pos, const int32_t* max_len, const int32_t* finished, int32_t* rb_q,
    int32_t* active, unsigned int* ctl, int32_t* out_len, int32_t* out_acc,
    int32_t* out_tokens, float* out_norm, unsigned long long* out_z, uint32_t* dev_err) {
    using Scan = cub::BlockScan<int, PLAN_NT>;
    __shared__ typename Scan::TempStorage tmp;
    const int tid = threadIdx.x;
    const int per = (n + PLAN_NT - 1) / PLAN_NT;
    const int b0 = min(n, tid * per), b1 = min(n, b0 + per);
    const int kp1 = k + 1;
    int mine = 0;
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
        mine += (q >= 0) ? 1 : 0;
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
    int excl, total;
    Scan(tmp).ExclusiveSum(mine, excl, total);
    for (int b = b0; b < b1; ++b)
        if (rb_q[b] >= 0) active[excl++] = b;
    if (tid == 0) {
        ctl[VCTL_NEXT] = 0u;
        ctl[VCTL_NACTIVE] = (unsigned)total;
    }
}

// Slice size limit (bytes per smem buffer; env BS_VERIFY_SLICE_KB overrides): small
// slices -> bigger clusters -> more resident CTAs per SM to hide each other's latencies.
static int slice_limit_bytes() {
    static int lim = 0;
    if (!lim) {
        const char* e = getenv("BS_VERIFY_SLICE_KB");
        lim = (e && atoi(e) > 0) ? atoi(e) * 1024 : 20 * 1024;
    }
    return lim;
}

static int pick_cluster(int V) {
    int C = 1;
    while (C < MAXC && (int64_t)((V + C - 1) / C) * 2 > slice_limit_bytes()) C <<= 1;
    return C;
}

template <int NT, int MINB>
static cudaError_t launch_rows(const VerifyArgs& a, int num_sms, int n, cudaStream_t st) {
    const size_t smem = (size_t)a.ntiles * 1024 + sizeof(VShared);
    static int configured = 0;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(verify_rows_kernel<NT, MINB>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(verify_rows_kernel<NT, MINB>,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        configured = 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)a.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // persistent grid: every resident cluster slot, but no more clusters than rollouts / 2
    static int max_clusters = 0;
    static size_t max_for_smem = 0;
    static int max_for_c = 0;
    if (max_clusters == 0 || max_for_smem != smem || max_for_c != a.C) {
        cfg.gridDim = dim3((unsigned)(a.C * num_sms), 1, 1);
        int mc = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&mc, verify_rows_kernel<NT, MINB>, &cfg);
        if (e != cudaSuccess || mc < 1) {
            cudaGetLastError();
            mc = std::max(1, num_sms / a.C);
        }
        max_clusters = mc;
        max_for_smem = smem;
        max_for_c = a.C;
    }
    const int clusters = std::max(1, std::min(max_clusters, (n + 1) / 2));
    cfg.gridDim = dim3((unsigned)(clusters * a.C), 1, 1);
    return cudaLaunchKernelEx(&cfg, verify_rows_kernel<NT, MINB>, a);
}

cudaError_t launch_verify(bs_ctx* ctx, int32_t n, const int32_t* slots, const void* logits,
                          const int64_t* row_index, int64_t stride, const int32_t* draft,
                          const int32_t* draft_len, int32_t k, float T, float top_p,
                          int32_t* out_tokens, int32_t* out_len, int32_t* out_acc,
                          float* out_norm, unsigned long long* out_z, cudaStream_t st) {
    (void)top_p;
    if (n == 0) return cudaSuccess;
    const int V = ctx->cfg.vocab;
    verify_plan_kernel<<<1, PLAN_NT, 0, st>>>(n, k, V, slots, draft, draft_len, ctx->pos.p,
                                              ctx->max_len.p, ctx->finished.p, ctx->rb_q.p,
                                              ctx->vqueue.p, ctx->vctl.p, out_len, out_acc,
                                              out_tokens, out_norm, out_z, ctx->dev_err.p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    VerifyArgs a = {};
    a.slots = slots;
    a.logits = static_cast<const uint16_t*>(logits);
    a.row_index = row_index;
    a.stride = stride;
    a.draft = draft;
    a.k = k;
    a.V = V;
    a.C = pick_cluster(V);
    a.SL = (((V + a.C - 1) / a.C) + 7) & ~7;
    a.ntiles = (a.SL + 255) / 256;
    a.S = ctx->S;
    a.eos = ctx->cfg.eos_id;
    a.T = T;
    a.c = (T > 0.f) ? (float)(1.4426950408889634 / (double)T) : 0.f;
    a.seed = ctx->cfg.seed;
    a.pos = ctx->pos.p;
    a.uid = ctx->uid.p;
    a.rb_q = ctx->rb_q.p;
    a.active = ctx->vqueue.p;
    a.ctl = ctx->vctl.p;
    a.dev_err = ctx->dev_err.p;
    a.out_tokens = out_tokens;
    a.out_len = out_len;
    a.out_acc = out_acc;
    a.out_norm = out_norm;
    a.out_z = out_z;
    a.stats = ctx->stats.p;
    if (a.SL >= 4096) {
        if ((size_t)a.ntiles * 1024 + sizeof(VShared) <= 72 * 1024)
            return launch_rows<256, 3>(a, ctx->num_sms, n, st);  // three CTAs per SM
        return launch_rows<256, 2>(a, ctx->num_sms, n, st);
    }
    return launch_rows<128, 4>(a, ctx->num_sms, n, st);
}

}  // namespace bs

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
