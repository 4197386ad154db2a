// verify.cu — fused vocab-row verify + resample (Eq. 2, Eq. 3 P:208-210,
// Alg. 1, bonus token P:308) for sm_100a.
//
// Kernel K3.  A PERSISTENT grid of thread-block clusters; a cluster of C
// CTAs owns one logits row at a time, CTA `rank` the vocabulary slice
// [rank*SL, (rank+1)*SL).  Work is claimed per ROLLOUT (one atomic each) and a rollout's
// rows are verified in Alg. 1's order, lazily: row j+1 is read only if row j accepted
// d_{j+1} (rows after the first rejection are never read).  Each cluster keeps two
// rollouts in flight and alternates between them, so while one row is computed the next
// row of the other rollout streams in (1-D bulk async copies on the TMA engine, mbarrier
// completion, L2 evict-first) — the dependency chain of one rollout never stalls the SM.
// Per row:
//   * pass 1: NaN-propagating bf16x2 max; every CTA pushes its slice max into all CTAs'
//     shared memory (DSMEM stores) -> cluster barrier -> row max;
//   * pass 2: integer masses of reading R with packed FFMA2/FADD2, exact u64 sums; slice
//     sums and mass(d) pushed over DSMEM -> cluster barrier -> Z, accept (Philox counter
//     (pos+j, ACCEPT), drawn while the row streams in);
//   * a residual / bonus sample only when needed: the CTA holding the CDF crossing
//     rescans the crossing warp's 256-element tiles and finalizes the rollout itself.
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "ctx.h"
#include "ptx.cuh"

namespace cg = cooperative_groups;

namespace bs {

constexpr int MAXC = 8;  // max cluster size

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

struct __align__(16) VShared {
    uint64_t full[2];  // TMA completion barrier per slot buffer
    // written remotely by every CTA of the cluster (index = source rank)
    float xmax[MAXC];
    uint32_t xbad[MAXC];
    int32_t xfirst[MAXC];
    unsigned long long xsum[MAXC];
    unsigned long long xmassd[MAXC];
    int32_t spare;  // claimed-ahead rollout index (written by the leader into all CTAs)
    // CTA-local
    float wmax[32];
    uint32_t wbad[32];
    int32_t wfirst[32];
    unsigned long long wsum[32];
    uint32_t racc[4], rsmp[4];  // Philox draws of the current row
    float m;
    int32_t ok;
    int32_t accept;
    int32_t need_sample;
    int32_t cross_rank;
    int32_t wstar;
    int32_t greedy;
    int32_t pad;
    unsigned long long z;
    unsigned long long ulocal;
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
__device__ __forceinline__ const uint16_t* row_ptr(const VerifyArgs& a, int b, int j) {
    const int kp1 = a.k + 1;
    const int64_t rowno = a.row_index ? a.row_index[(int64_t)b * kp1 + j] : (int64_t)b * kp1 + j;
    return a.logits + rowno * a.stride;
}

// Issue the bulk copy of this CTA's slice of row (b, j) into `buf` (elected thread).
__device__ __forceinline__ void issue_load(const VerifyArgs& a, int b, int j, int rank,
                                           uint16_t* buf, uint64_t* bar, uint64_t pol) {
    const int s0 = rank * a.SL, s1 = min(a.V, s0 + a.SL);
    const int len = max(0, s1 - s0);
    const uint16_t* src = row_ptr(a, b, j) + s0;
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

template <int NT>
__global__ void __launch_bounds__(NT) verify_rows_kernel(const VerifyArgs a) {
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

    if (tid == 0) {
        mbar_init(&sh.full[0], 1);
        mbar_init(&sh.full[1], 1);
        fence_mbar_init();
    }
    for (int i = tid; i < STAT_COUNT; i += NT) sh.stat[i] = 0ull;
    // -inf padding beyond the slice (never written by the bulk copies)
    for (int e = len + tid; e < a.ntiles * 256; e += NT) {
        bufs[0][e] = (uint16_t)0xFF80u;
        bufs[1][e] = (uint16_t)0xFF80u;
    }
    if (rank == 0 && tid == 0) {  // claim two rollouts + one spare
        const int base = (int)atomicAdd(a.ctl + VCTL_NEXT, 3u);
        for (int rr = 0; rr < C; ++rr) {
            VShared* o = cluster.map_shared_rank(&sh, rr);
            o->xfirst[0] = base;  // scratch for the broadcast below
        }
    }
    __syncthreads();
    cluster.sync();
    const int base0 = sh.xfirst[0];
    int rb[2], rj[2];  // rollout (index into active[], -1 = empty) and row of each slot
    rb[0] = (base0 < nact) ? base0 : -1;
    rb[1] = (base0 + 1 < nact) ? base0 + 1 : -1;
    int spare = (base0 + 2 < nact) ? base0 + 2 : -1;
    bool exhausted = (base0 + 2 >= nact - 1);
    rj[0] = rj[1] = 0;
    if (tid == 0) {
        for (int sl = 0; sl < 2; ++sl)
            if (rb[sl] >= 0) issue_load(a, a.active[rb[sl]], 0, rank, bufs[sl], &sh.full[sl], pol);
    }
    uint32_t ph[2] = {0u, 0u};
    int cur = 0;
    if (rb[0] < 0) cur = 1;

    while (rb[0] >= 0 || rb[1] >= 0) {
        if (rb[cur] < 0) cur ^= 1;
        const int b = a.active[rb[cur]];
        const int j = rj[cur];
        const int q = a.rb_q[b];
        const int slot = a.slots[b];
        uint16_t* sl = bufs[cur];
        const int d = (j < q) ? a.draft[(int64_t)b * a.k + j] : -1;  // d_{j+1}, tested on row j
        // leader claims the next spare early; the atomic's latency overlaps pass 1
        int claimed = -1;
        const bool want_spare = (rank == 0 && tid == 0 && spare < 0 && !exhausted);
        if (want_spare) claimed = (int)atomicAdd(a.ctl + VCTL_NEXT, 1u);
        // the row's two Philox draws, while the slice streams in
        if (tid == 32) {
            const uint64_t uidv = a.uid[slot];
            const uint32_t position = (uint32_t)(a.pos[slot] + j);
            const U128 r1 = draw(a.seed, uidv, position, PURPOSE_ACCEPT);
            const U128 r2 = draw(a.seed, uidv, position, PURPOSE_SAMPLE);
            sh.racc[0] = r1.x0; sh.racc[1] = r1.x1; sh.racc[2] = r1.x2; sh.racc[3] = r1.x3;
            sh.rsmp[0] = r2.x0; sh.rsmp[1] = r2.x1; sh.rsmp[2] = r2.x2; sh.rsmp[3] = r2.x3;
        }
        mbar_wait(&sh.full[cur], ph[cur]);
        ph[cur] ^= 1u;
        {   // ragged part (unaligned rows or a slice length not a multiple of 8)
            const uint16_t* src = row_ptr(a, b, j) + s0;
            const bool aligned = ((reinterpret_cast<uintptr_t>(src) & 15u) == 0);
            const int bulk = aligned ? (len & ~7) : 0;
            if (bulk < len) {
                for (int e = bulk + tid; e < len; e += NT) sl[e] = src[e];
                __syncthreads();
            }
        }
        // ---- pass 1: max (NaN-propagating on bf16x2)
        {
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
            if (tid < C) {  // push this slice's max into CTA `tid`
                float mloc = -INFINITY;
                uint32_t bb = 0;
                for (int w = 0; w < NW; ++w) {
                    mloc = fmaxf(mloc, sh.wmax[w]);
                    bb |= sh.wbad[w];
                }
                VShared* o = cluster.map_shared_rank(&sh, tid);
                o->xmax[rank] = mloc;
                o->xbad[rank] = bb;
            }
            if (want_spare) {
                for (int rr = 0; rr < C; ++rr) cluster.map_shared_rank(&sh, rr)->spare = claimed;
            }
        }
        cluster.sync();  // #1: slice maxima (and a claimed spare) visible everywhere
        if (tid == 0) {
            float m = -INFINITY;
            uint32_t bb = 0;
            for (int rr = 0; rr < C; ++rr) {
                m = fmaxf(m, sh.xmax[rr]);
                bb |= sh.xbad[rr];
            }
            int ok = 1;
            uint32_t err = 0;
            if (bb) { ok = 0; err |= DEV_BAD_LOGIT; }
            else if (m == -INFINITY) { ok = 0; err |= DEV_ALL_NEGINF; }
            else if (a.T > 0.f && !(fabsf(__fmul_rn(m, a.c)) < 16777216.0f)) { ok = 0; err |= DEV_RANGE; }
            if (err && rank == 0) atomicOr(a.dev_err, err);
            sh.m = m;
            sh.ok = ok;
        }
        if (spare < 0 && !exhausted) {  // uniform: everyone read the broadcast spare
            const int cl = sh.spare;
            if (cl < nact) spare = cl;
            if (cl >= nact - 1) exhausted = true;
        }
        __syncthreads();
        const float m = sh.m;
        const bool ok = sh.ok != 0;
        bool finished_here = false;  // this rollout's step is decided at row j
        bool accepted = false;
        MassParams mp;
        if (a.T == 0.f) {
            // ---- greedy (R1): first index attaining the max
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
            if (lane == 0) sh.wfirst[warp] = first;
            __syncthreads();
            if (tid < C) {
                int f = 0x7FFFFFFF;
                for (int w = 0; w < NW; ++w) f = min(f, sh.wfirst[w]);
                cluster.map_shared_rank(&sh, tid)->xfirst[rank] = (f == 0x7FFFFFFF) ? f : s0 + f;
            }
            cluster.sync();  // #2
            if (tid == 0) {
                int g = 0x7FFFFFFF;
                for (int rr = 0; rr < C; ++rr) g = min(g, sh.xfirst[rr]);
                sh.greedy = ok ? g : -1;
                sh.accept = (ok && j < q && d == g) ? 1 : 0;
                sh.z = 1ull;
                sh.need_sample = 0;
            }
            __syncthreads();
            accepted = sh.accept != 0;
            if (rank == 0 && tid == 0) {
                if (a.out_norm) a.out_norm[(int64_t)b * kp1 + j] = ok ? 1.0f : 0.f;
                if (a.out_z) a.out_z[(int64_t)b * kp1 + j] = ok ? 1ull : 0ull;
            }
            const bool eos_acc = accepted && a.eos >= 0 && d == a.eos;
            finished_here = !accepted || eos_acc;
            if (finished_here && rank == 0 && tid == 0)
                finalize_rollout(a, sh, b, j, q, eos_acc, sh.greedy);
        } else {
            // ---- pass 2: integer masses (R2-R4), exact sums
            mp.c = a.c;
            mp.nmc = -__fmul_rn(m, a.c);
            mp.clampv = -(float)(a.S + 2);
            mp.magic = 12582912.0f + (float)a.S;
            uint64_t acc = 0;
            if (ok) {
                for (int t = t0; t < t1; ++t) acc += mass8(lds128(sl + t * 256 + lane * 8), mp);
            }
            acc = warp_sum_u64(acc);
            if (lane == 0) sh.wsum[warp] = acc;
            __syncthreads();
            if (tid < C) {
                uint64_t sum = 0;
                for (int w = 0; w < NW; ++w) sum += sh.wsum[w];
                const uint64_t md = (ok && d >= s0 && d < s1) ? mass_of(bf16_at(sl, d - s0), mp) : 0ull;
                VShared* o = cluster.map_shared_rank(&sh, tid);
                o->xsum[rank] = sum;
                o->xmassd[rank] = md;
            }
            cluster.sync();  // #2: slice sums visible everywhere
            if (tid == 0) {
                uint64_t Zs = 0, md = 0;
                for (int rr = 0; rr < C; ++rr) {
                    Zs += sh.xsum[rr];
                    md += sh.xmassd[rr];
                }
                int accept = 0, need = 1;
                if (ok && j < q) {
                    const U128 r1{sh.racc[0], sh.racc[1], sh.racc[2], sh.racc[3]};
                    accept = (uniform_floor(r1, Zs) < md) ? 1 : 0;
                    need = !accept;
                }
                const int excl = (j < q) ? d : -1;
                int cross = -1;
                uint64_t ulocal = 0;
                if (ok && need) {
                    const U128 r2{sh.rsmp[0], sh.rsmp[1], sh.rsmp[2], sh.rsmp[3]};
                    const uint64_t U2 = uniform_floor(r2, Zs - ((j < q) ? md : 0ull));
                    uint64_t before = 0;
                    for (int rr = 0; rr < C; ++rr) {
                        const int r0 = rr * a.SL, r1e = min(a.V, r0 + a.SL);
                        const uint64_t adj = sh.xsum[rr] - ((excl >= r0 && excl < r1e) ? md : 0ull);
                        if (U2 < before + adj) {
                            cross = rr;
                            ulocal = U2 - before;
                            break;
                        }
                        before += adj;
                    }
                }
                sh.z = Zs;
                sh.accept = accept;
                sh.need_sample = (ok && need) ? 1 : 0;
                sh.cross_rank = cross;
                sh.wstar = -1;
                if (cross == rank) {
                    uint64_t before = 0;
                    const int span = tpw * 256;
                    for (int w = 0; w < NW; ++w) {
                        const int w0 = s0 + w * span, w1 = min(s1, w0 + span);
                        const uint64_t adj = sh.wsum[w] - ((excl >= w0 && excl < w1) ? md : 0ull);
                        if (ulocal < before + adj) {
                            sh.wstar = w;
                            sh.ulocal = ulocal - before;
                            break;
                        }
                        before += adj;
                    }
                }
                if (rank == 0) {
                    const uint64_t Zo = ok ? Zs : 0ull;
                    if (a.out_norm) a.out_norm[(int64_t)b * kp1 + j] = ok ? (float)ldexp((double)Zo, -a.S) : 0.f;
                    if (a.out_z) a.out_z[(int64_t)b * kp1 + j] = Zo;
                }
            }
            __syncthreads();
            accepted = ok && sh.accept;
            const bool eos_acc = accepted && a.eos >= 0 && d == a.eos;
            finished_here = !accepted || eos_acc;
            if (finished_here) {
                if (!ok) {
                    if (rank == 0 && tid == 0) finalize_rollout(a, sh, b, j, q, false, -1);
                } else if (eos_acc) {
                    if (rank == 0 && tid == 0) finalize_rollout(a, sh, b, j, q, true, -1);
                } else if (sh.cross_rank == rank && warp == sh.wstar) {
                    // ---- residual / bonus sample: rescan the crossing warp's tiles (R8)
                    const int excl = (j < q) ? d : -1;
                    const uint64_t U = sh.ulocal;
                    uint64_t run = 0;
                    for (int t = t0; t < t1; ++t) {
                        const int e0 = t * 256 + lane * 8;
                        const uint4 v = lds128(sl + e0);
                        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
                        uint64_t mm[8];
#pragma unroll
                        for (int i = 0; i < 4; ++i) mass_pair(w4[i], mp, mm[2 * i], mm[2 * i + 1]);
                        uint64_t ls = 0;
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            if (s0 + e0 + i == excl) mm[i] = 0;
                            ls += mm[i];
                        }
                        const uint64_t incl = warp_incl_scan_u64(ls, lane);
                        const uint64_t tot = shfl_u64(incl, 31);
                        if (U < run + tot) {
                            const unsigned hit = __ballot_sync(0xFFFFFFFFu, U < run + incl);
                            const int L = __ffs(hit) - 1;
                            if (lane == L) {
                                uint64_t cum = run + incl - ls;
                                int tok = -1;
#pragma unroll
                                for (int i = 0; i < 8; ++i) {
                                    cum += mm[i];
                                    if (tok < 0 && cum > U) tok = s0 + e0 + i;
                                }
                                finalize_rollout(a, sh, b, j, q, false, tok);
                            }
                            break;
                        }
                        run += tot;
                    }
                }
            }
        }
        // ---- advance this slot: next row of the same rollout, or a new rollout
        __syncthreads();  // the sampling warp is done reading bufs[cur]
        if (!finished_here) {
            rj[cur] = j + 1;
            if (tid == 0) issue_load(a, b, j + 1, rank, bufs[cur], &sh.full[cur], pol);
        } else {
            rb[cur] = spare;
            rj[cur] = 0;
            spare = -1;
            if (rb[cur] >= 0 && tid == 0)
                issue_load(a, a.active[rb[cur]], 0, rank, bufs[cur], &sh.full[cur], pol);
        }
        cur ^= 1;
    }
    // flush the CTA's statistics counters
    __syncthreads();
    if (a.stats)
        for (int i = tid; i < STAT_COUNT; i += NT)
            if (sh.stat[i]) atomicAdd(a.stats + i, sh.stat[i]);
    cluster.sync();  // no CTA exits while a peer may still write into its shared memory
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

static int pick_cluster(int V) {
    // two slice buffers of <= ~40 KB: two CTAs per SM overlap each other's barriers
    int C = 1;
    while (C < MAXC && (int64_t)((V + C - 1) / C) * 2 > 40 * 1024) C <<= 1;
    return C;
}

template <int NT>
static cudaError_t launch_rows(const VerifyArgs& a, int num_sms, int n, cudaStream_t st) {
    const size_t smem = (size_t)a.ntiles * 1024 + sizeof(VShared);
    static int configured = 0;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(verify_rows_kernel<NT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
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
    if (max_clusters == 0 || max_for_smem != smem) {
        cfg.gridDim = dim3((unsigned)(a.C * num_sms), 1, 1);
        int mc = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&mc, verify_rows_kernel<NT>, &cfg);
        if (e != cudaSuccess || mc < 1) {
            cudaGetLastError();
            mc = std::max(1, num_sms / a.C);
        }
        max_clusters = mc;
        max_for_smem = smem;
    }
    const int clusters = std::max(1, std::min(max_clusters, (n + 1) / 2));
    cfg.gridDim = dim3((unsigned)(clusters * a.C), 1, 1);
    return cudaLaunchKernelEx(&cfg, verify_rows_kernel<NT>, a);
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
    if (a.SL >= 4096) return launch_rows<256>(a, ctx->num_sms, n, st);
    return launch_rows<128>(a, ctx->num_sms, n, st);
}

}  // namespace bs
