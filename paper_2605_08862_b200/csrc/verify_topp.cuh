// verify_topp.cuh — verify + resample under top-k / top-p filtering (readings R5k, R5,
// DESIGN.md §2/§4), included by verify.cu (shares its row queue, descriptors and completion
// protocol).
//
// Top-k (R5k, applied first) keeps {i : mass_i >= tau_k}, tau_k the top_k-th largest
// mass: mass is nondecreasing in the logit, so tau_k = mass(kappa), kappa the top_k-th largest
// 16-bit order key among the positive-mass tokens, found by a COUNT-weighted select over the
// same coarse bins (pass 2 also counts tokens per bin; pass 3k counts the 16 keys of the
// crossing bin); the kept sum Z_k comes from one filtered tile pass.  Top-p then runs on the
// top-k masses (Theta from Z_k); its crossing key lies among keys with mass >= tau_k because
// Theta <= Z_k, so the unfiltered mass histograms still locate it.
//
// The tie-closed nucleus keeps {i : mass_i >= tau}, tau = max{t : F(t) >= Theta},
// F(t) = sum of the masses >= t.  mass is a nondecreasing function of the bf16 logit, so
// tau is found by a mass-weighted select over the 16-bit order key of the logits instead
// of a sort:
//   pass 1  row max (R1, validity R0);
//   pass 2  masses: Z, and the mass of each of 4096 coarse key bins (key >> 4);
//   select  the coarse bin B where the descending cumulative mass reaches Theta;
//   pass 3  the masses of the 16 keys inside B -> the crossing key k*, tau = mass(k*);
//   pass 4  (only when a sample is drawn, or when keys below k* share its mass) the
//           filtered masses' 256-element tile sums, which give Z' and the inverse CDF.
// Each row is split over an 8-CTA thread-block cluster (CTA r: elements [r SL, r SL + SL)):
// the slice is staged in shared memory by one bulk copy (when it fits beside the histograms at
// two CTAs per SM; else the passes stream it from L2), every pass runs on the slices in
// parallel, the per-slice histograms and sums are added into the leader CTA's shared memory
// over DSMEM (remote shared atomics) at cluster barriers, and every CTA then gathers the
// cluster totals from the leader into its own shared memory (a few threads), so all of them
// take the same decisions; the sample's crossing slice rescans its crossing tile.  (One CTA per row, the
// round-1 layout, made a tail step of the long-context config cost ~150 us per row.)
#pragma once
// (included inside namespace bs)

constexpr int TP_CL = 8;              // CTAs per row (cluster)
constexpr int TP_NT = 512;            // threads
constexpr int TP_NW = TP_NT / 32;     // warps
constexpr int TP_H1 = 4096;           // coarse key bins
constexpr int TP_MAXLT = 256;         // 256-element tiles per slice: V <= 8 * 65536 = 524288
constexpr int TP_MAXT = TP_CL * TP_MAXLT;

struct TopPShared {
    uint32_t h1lo[TP_H1], h1hi[TP_H1];  // coarse-bin masses (Hist64); the leader's: cluster sums
    uint32_t hc[TP_H1];                 // top-k: positive-mass tokens per coarse bin
    uint32_t h2c[16];                   // top-k: positive-mass tokens per key of the crossing bin
    unsigned long long h2part[TP_CL][16];  // the leader's: each slice's masses of the 16 keys of
                                           // the crossing bin (plain remote stores, no atomics)
    uint32_t h3c[16];                   // top-p: tokens per key of the crossing bin (this slice)
    unsigned long long tsum[TP_MAXLT];  // this slice's 256-element tile sums
    unsigned long long stat[STAT_COUNT];
    float wmax[TP_NW];
    uint32_t wbad[TP_NW];
    // written into the LEADER's copy by every CTA (DSMEM), read by all after a cluster barrier
    float cmax[TP_CL];
    uint32_t cbad[TP_CL];
    unsigned long long zsum[TP_CL];     // slice sums: unfiltered
    unsigned long long fsum[3][TP_CL];  // slice sums of filtered passes (rotating)
    int32_t cand;                       // the sampled token (from the crossing slice)
    // the leader's broadcasts
    RowDesc dsc;
    unsigned long long bz[2];  // [0] Theta remaining inside the coarse bin, [1] sum above it
    int32_t bsel;              // coarse bin B
    int32_t bselk, needk;      // top-k: coarse bin of kappa, tokens still needed inside it
    uint64_t sbar;             // the staged slice's bulk copy (mbarrier)
    // this CTA's copies of the leader's cluster totals, gathered by a few threads right after the
    // barrier that completes them (every thread re-reading them over DSMEM, in loops that break
    // early, cost serial remote round trips under 4,096-fold contention)
    float xm[TP_CL];
    uint32_t xb[TP_CL];
    unsigned long long xz[TP_CL];   // the current slice sums (tiles_sums)
    unsigned long long xh2[16];     // the crossing bin's key masses
    unsigned long long xbz[2];
    uint32_t xc[16];                // top-k: the crossing bin's key counts
    RowDesc xdsc;                   // the row's descriptor
    int32_t xB;                     // the coarse bin of the top-p crossing
    unsigned long long wtot[TP_NW];  // coarse select: per-warp mass totals (block scan)
};

// The slice is staged in shared memory (one bulk copy per row, after the TopPShared block) when
// both fit two CTAs per SM; the passes then read shared memory instead of re-streaming L2.
__host__ __device__ constexpr size_t tp_shared_bytes() { return (sizeof(TopPShared) + 127) & ~size_t(127); }
constexpr size_t TP_STAGE_MAX = 110 * 1024;  // per CTA, two CTAs per SM

// Order-preserving map of bf16 bit patterns to 16-bit keys (larger value -> larger key).
__device__ __forceinline__ uint32_t tp_key(uint32_t b) {
    return (b & 0x8000u) ? (~b & 0xFFFFu) : (b | 0x8000u);
}
__device__ __forceinline__ uint32_t tp_unkey(uint32_t k) {
    return (k & 0x8000u) ? (k & 0x7FFFu) : (~k & 0xFFFFu);
}

// Shared-memory 64-bit histogram bins kept as two 32-bit words: an add is one native 32-bit
// shared atomic on the low word plus, only when it carries or the value has high bits, one on the
// high word (a 64-bit shared atomic add is far slower under contention).
struct Hist64 {
    uint32_t* lo;
    uint32_t* hi;
    __device__ __forceinline__ void add(uint32_t bin, uint64_t v) const {
        const uint32_t vl = (uint32_t)v;
        const uint32_t old = atomicAdd(lo + bin, vl);
        const uint32_t h = (uint32_t)(v >> 32) + ((old + vl < old) ? 1u : 0u);
        if (h) atomicAdd(hi + bin, h);
    }
    __device__ __forceinline__ uint64_t get(int bin) const { return ((uint64_t)hi[bin] << 32) | lo[bin]; }
    __device__ __forceinline__ void clear(int bin) const {
        lo[bin] = 0u;
        hi[bin] = 0u;
    }
};

// Lane's 8 consecutive logits of tile t (-inf beyond V / scalar path when unaligned).
__device__ __forceinline__ uint4 tp_load8(const uint16_t* row, int e0, int V, bool aligned) {
    if (aligned && e0 + 8 <= V) return __ldcg(reinterpret_cast<const uint4*>(row + e0));
    uint16_t t8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) t8[i] = (e0 + i < V) ? row[e0 + i] : (uint16_t)0xFF80u;
    return make_uint4(t8[0] | ((uint32_t)t8[1] << 16), t8[2] | ((uint32_t)t8[3] << 16),
                      t8[4] | ((uint32_t)t8[5] << 16), t8[6] | ((uint32_t)t8[7] << 16));
}
__device__ __forceinline__ void tp_unpack(const uint4 v, uint32_t b[8]) {
    b[0] = v.x & 0xFFFFu; b[1] = v.x >> 16; b[2] = v.y & 0xFFFFu; b[3] = v.y >> 16;
    b[4] = v.z & 0xFFFFu; b[5] = v.z >> 16; b[6] = v.w & 0xFFFFu; b[7] = v.w >> 16;
}

// Stream the slice tile by tile (warp w: tiles w, w + TP_NW, ...), TP_U tiles' loads issued
// before any is consumed (from the staged copy in shared memory, or from L2 when the slice was
// too large to stage).
#ifndef BS_TP_U
#define BS_TP_U 2
#endif
constexpr int TP_U = BS_TP_U;
// sbuf (staged slice, -inf padded to whole tiles) replaces the global loads when non-null.
template <class F>
__device__ __forceinline__ void tp_stream(const uint16_t* row, const uint16_t* sbuf, int ntile, int V, bool aligned,
                                          int warp, int lane, F&& f) {
    for (int t0 = warp; t0 < ntile; t0 += TP_NW * TP_U) {
        uint4 v[TP_U];
#pragma unroll
        for (int u = 0; u < TP_U; ++u) {
            const int t = t0 + u * TP_NW;
            v[u] = (t < ntile) ? (sbuf ? lds128(sbuf + t * 256 + lane * 8) : tp_load8(row, t * 256 + lane * 8, V, aligned))
                               : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
        }
#pragma unroll
        for (int u = 0; u < TP_U; ++u) {
            const int t = t0 + u * TP_NW;
            if (t < ntile) f(t, v[u]);  // (warp-uniform)
        }
    }
}

// Counts of the 16 keys of coarse bin B in this thread's elements of the slice, 8 bits per key
// packed in 4 words (a thread sees at most 128 elements per pass: SL <= 65536 over 512 threads).
// Every element with a given key has the same mass (mass is a function of the bf16 value), so a
// key's mass total is its count times that mass: no per-element 64-bit shared atomics, which
// all landed on the same 16 bins.
__device__ __forceinline__ void tp_key_count(uint32_t c4[4], uint32_t kk, int B) {
    if ((int)(kk >> 4) == B) {
        const uint32_t k4 = kk & 15u, w = k4 >> 2, inc = 1u << ((k4 & 3u) * 8u);
        c4[0] += (w == 0u) ? inc : 0u;
        c4[1] += (w == 1u) ? inc : 0u;
        c4[2] += (w == 2u) ? inc : 0u;
        c4[3] += (w == 3u) ? inc : 0u;
    }
}
// The warp's count of key kq of the packed per-lane counts.
__device__ __forceinline__ uint32_t tp_warp_count(const uint32_t c4[4], int kq) {
    return __reduce_add_sync(0xFFFFFFFFu, (c4[kq >> 2] >> ((kq & 3) * 8)) & 0xFFu);
}

__global__ void __cluster_dims__(TP_CL, 1, 1) __launch_bounds__(TP_NT, 2)
verify_topp_kernel(const VerifyArgs a, float top_p, int top_k, int SL, int staged) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(128) uint8_t tp_smem[];
    TopPShared& sh = *reinterpret_cast<TopPShared*>(tp_smem);
    uint16_t* const sbuf_base = reinterpret_cast<uint16_t*>(tp_smem + tp_shared_bytes());
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    TopPShared* L = cl.map_shared_rank(&sh, 0);  // the leader's copy
    pdl_wait();  // dependents launch at exit (the cluster kernel plans before its wait)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef BS_PHASE_TIMING
    long long ph_t = clock64();
#endif
    const int rows = (int)a.ctl[VCTL_ROWS];
    const int V = a.V;
    const int e_lo = rank * SL, len = max(0, min(SL, V - e_lo));
    const int nlt = (len + 255) / 256;  // this slice's tiles
    const uint64_t P = (uint64_t)llround((double)top_p * 4294967296.0);  // R5 (top_p < 1)
    const bool use_p = top_p < 1.f, use_k = top_k > 0;
    for (int i = tid; i < STAT_COUNT; i += TP_NT) sh.stat[i] = 0ull;
    if (tid == 0) mbar_init(&sh.sbar, 1);
    __syncthreads();
    uint32_t sphase = 0;  // the staging barrier's phase
    const Hist64 H1{sh.h1lo, sh.h1hi};
    const Hist64 H1L{L->h1lo, L->h1hi};

    for (;;) {
        if (rank == 0 && tid == 0) sh.dsc = claim_row(a, rows);
        // clear this CTA's accumulators (the leader's are the cluster totals)
        for (int i = tid; i < TP_H1; i += TP_NT) {
            H1.clear(i);
            sh.hc[i] = 0u;
        }
        if (tid < 16) {
            sh.h2c[tid] = 0u;
            sh.h3c[tid] = 0u;
        }
        PH_MARK(0); cl.sync(); PH_MARK(8);  // S1: the claim is published; every accumulator is clear; the last row is done
        static_assert(sizeof(RowDesc) == 48, "RowDesc layout");
        if (tid < 12) reinterpret_cast<uint32_t*>(&sh.xdsc)[tid] = reinterpret_cast<const uint32_t*>(&L->dsc)[tid];
        __syncthreads();
        const RowDesc dsc = sh.xdsc;
        if (dsc.b < 0) {
            cl.sync();  // no CTA may exit while another still reads the leader's shared memory
            break;
        }
        const uint16_t* row = a.logits + dsc.rowno * a.stride;
        const uint16_t* srow = row + e_lo;
        const bool aligned = dsc.aligned != 0;
        const int j = dsc.j, q = dsc.q, d = dsc.d;
        const uint16_t* sbuf = nullptr;
        if (staged) {  // the slice into shared memory: one bulk copy, -inf padding to whole tiles
            const int ncopy = aligned ? (len & ~7) : 0;  // a 16-byte multiple
            if (tid == 0) {
                if (ncopy) {
                    fence_proxy_async_smem();  // the previous row's reads of the buffer come first
                    mbar_arrive_expect_tx(&sh.sbar, (uint32_t)ncopy * 2u);
                    bulk_g2s(sbuf_base, srow, (uint32_t)ncopy * 2u, &sh.sbar, policy_evict_first());
                } else {
                    mbar_arrive(&sh.sbar);
                }
            }
            for (int e = ncopy + tid; e < nlt * 256; e += TP_NT) sbuf_base[e] = (e < len) ? srow[e] : (uint16_t)0xFF80u;
            mbar_wait(&sh.sbar, sphase);
            sphase ^= 1u;
            __syncthreads();  // the generic tail fill
            sbuf = sbuf_base;
        }

        // ---------------------------------------------------- pass 1: max (slice, then cluster)
        uint32_t mx = 0xFF80FF80u;
        tp_stream(srow, sbuf, nlt, len, aligned, warp, lane, [&](int, const uint4 v) {
            mx = hmax2_nan_u32(mx, v.x);
            mx = hmax2_nan_u32(mx, v.y);
            mx = hmax2_nan_u32(mx, v.z);
            mx = hmax2_nan_u32(mx, v.w);
        });
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
        __syncthreads();
        if (tid == 0) {
            float cm = -INFINITY;
            uint32_t cb = 0;
            for (int w = 0; w < TP_NW; ++w) {
                cm = fmaxf(cm, sh.wmax[w]);
                cb |= sh.wbad[w];
            }
            L->cmax[rank] = cm;
            L->cbad[rank] = cb;
        }
        PH_MARK(1); cl.sync(); PH_MARK(9);  // S2: every slice's max in the leader
        if (tid < TP_CL) {
            sh.xm[tid] = L->cmax[tid];
            sh.xb[tid] = L->cbad[tid];
        }
        __syncthreads();
        float m = -INFINITY;
        uint32_t bb = 0;
        for (int r = 0; r < TP_CL; ++r) {
            m = fmaxf(m, sh.xm[r]);
            bb |= sh.xb[r];
        }
        uint32_t err = 0;
        if (bb) err |= DEV_BAD_LOGIT;
        else if (m == -INFINITY) err |= DEV_ALL_NEGINF;
        else if (!(fabsf(__fmul_rn(m, a.c)) < 16777216.0f)) err |= DEV_RANGE;
        if (err) {  // R0: the row is an error; the rollout stops (no token)
            if (rank == 0 && warp == 0) {  // reported at finalize only if Alg. 1 needs this row
                if (lane == 0) sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                int no = 0;
                int32_t tk = -1;
                complete_row_warp(a, sh.stat, dsc.b, j, q, ST_ERR, (int)err, 0ull, 0.f, lane, no, tk);
            }
            cl.sync();  // S_end: every CTA is done reading the leader's row state
            continue;
        }
        MassParams mp;
        mp.c = a.c;
        mp.nmc = -__fmul_rn(m, a.c);
        mp.clampv = -(float)(a.S + 2);
        mp.magic = 12582912.0f + (float)a.S;

        // ---------------------------------------------------- pass 2: masses, Z, coarse bins
        tp_stream(srow, sbuf, nlt, len, aligned, warp, lane, [&](int t, const uint4 v) {
            uint64_t mm[8];
            mass_pair(v.x, mp, mm[0], mm[1]);
            mass_pair(v.y, mp, mm[2], mm[3]);
            mass_pair(v.z, mp, mm[4], mm[5]);
            mass_pair(v.w, mp, mm[6], mm[7]);
            uint32_t bits[8];
            tp_unpack(v, bits);
            uint64_t s = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                s += mm[i];
                if (mm[i]) {
                    const uint32_t kb = tp_key(bits[i]) >> 4;
#ifndef BS_TP_EXP_NOHIST  // measurement only: pass 2 without its histogram atomics
                    if (use_p) H1.add(kb, mm[i]);
#else
                    (void)kb;
#endif
                    if (use_k) atomicAdd(&sh.hc[kb], 1u);
                }
            }
            const uint64_t ws = warp_sum_u51(s);
            if (lane == 0) sh.tsum[t] = ws;
        });
        __syncthreads();
        // this slice's tile sums -> its sum in the leader (every thread computes it, tid 0 stores)
        auto slice_total = [&]() {
            uint64_t zl = 0;
            for (int t = lane; t < nlt; t += 32) zl += sh.tsum[t];
            return warp_sum_u64(zl);
        };
        {
            const uint64_t zs = slice_total();
            if (tid == 0) L->zsum[rank] = zs;
        }
        if (rank != 0) {  // this slice's histograms into the leader's (remote shared atomics)
            for (int i = tid; i < TP_H1; i += TP_NT) {
                if (use_p) {
                    const uint64_t h = H1.get(i);
                    if (h) H1L.add((uint32_t)i, h);
                }
                if (use_k && sh.hc[i]) atomicAdd(&L->hc[i], sh.hc[i]);
            }
        }
        PH_MARK(2); cl.sync(); PH_MARK(10);  // S3: cluster histograms and slice sums in the leader
        if (tid < TP_CL) sh.xz[tid] = L->zsum[tid];
        __syncthreads();
        uint64_t Z = 0;
        for (int r = 0; r < TP_CL; ++r) Z += sh.xz[r];  // R4: the unfiltered normaliser
        // filtered slice tile sums (masses >= t) and their slice total into fsum[slot]
        uint64_t tiles_tau = 0;  // pass 2's tile sums keep every mass
        const unsigned long long* tiles_sums = sh.xz;  // (this CTA's copy of the slice sums)
        int fslot = 0;
        auto filtered_tiles = [&](uint64_t t) {
            __syncthreads();  // earlier readers of sh.tsum are done
            tp_stream(srow, sbuf, nlt, len, aligned, warp, lane, [&](int tt, const uint4 v) {
                uint64_t mm[8];
                mass_pair(v.x, mp, mm[0], mm[1]);
                mass_pair(v.y, mp, mm[2], mm[3]);
                mass_pair(v.z, mp, mm[4], mm[5]);
                mass_pair(v.w, mp, mm[6], mm[7]);
                uint64_t s = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) s += (mm[i] >= t) ? mm[i] : 0ull;
                const uint64_t ws = warp_sum_u51(s);
                if (lane == 0) sh.tsum[tt] = ws;
            });
            __syncthreads();
            const uint64_t fs = slice_total();
            if (tid == 0) L->fsum[fslot][rank] = fs;
            PH_MARK(3); cl.sync(); PH_MARK(11);  // every slice's filtered sum in the leader
            if (tid < TP_CL) sh.xz[tid] = L->fsum[fslot][tid];  // (readers of the previous copy are
            __syncthreads();                                      //  past this call's first barrier)
            tiles_tau = t;
            tiles_sums = sh.xz;
            fslot = (fslot + 1) % 3;
            uint64_t tot = 0;
            for (int r = 0; r < TP_CL; ++r) tot += tiles_sums[r];
            return tot;
        };
        // ---------------------------------------------------- top-k (R5k): tau_k, Z_k
        uint64_t tau = 0, Zk = Z;
        if (use_k) {
            if (rank == 0 && warp == 0) {  // count select over the coarse bins, heaviest first
                const int per = TP_H1 / 32;
                const int lo = (31 - lane) * per;
                uint32_t ls = 0;
                for (int i = 0; i < per; ++i) ls += sh.hc[lo + i];
                uint32_t incl = ls;
#pragma unroll
                for (int dd = 1; dd < 32; dd <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, incl, dd);
                    if (lane >= dd) incl += o;
                }
                const unsigned hit = __ballot_sync(0xFFFFFFFFu, incl >= (uint32_t)top_k);
                if (lane == 0 && !hit) sh.bselk = -1;  // fewer than top_k positive masses: keep all
                const int Lh = hit ? (__ffs(hit) - 1) : 32;
                if (lane == Lh) {
                    uint32_t above = incl - ls;
                    int Bk = lo;
                    for (int i = per - 1; i >= 0; --i) {
                        const uint32_t h = sh.hc[lo + i];
                        if (above + h >= (uint32_t)top_k) {
                            Bk = lo + i;
                            break;
                        }
                        above += h;
                    }
                    sh.bselk = Bk;
                    sh.needk = top_k - (int)above;
                }
            }
            cl.sync();  // S4: the leader's select
            const int Bk = L->bselk;
            if (Bk >= 0) {
                // pass 3k: counts of the 16 keys inside bin Bk (slice -> leader)
                uint32_t c4[4] = {0u, 0u, 0u, 0u};
                tp_stream(srow, sbuf, nlt, len, aligned, warp, lane, [&](int, const uint4 v) {
                    uint32_t bits[8];
                    tp_unpack(v, bits);
#pragma unroll
                    for (int i = 0; i < 8; ++i) tp_key_count(c4, tp_key(bits[i]), Bk);
                });
#pragma unroll
                for (int kq = 0; kq < 16; ++kq) {  // positive-mass tokens only (mass is the key's)
                    const uint32_t cnt = tp_warp_count(c4, kq);
                    if (lane == 0 && cnt &&
                        mass_of(__uint_as_float(tp_unkey((uint32_t)(Bk * 16 + kq)) << 16), mp))
                        atomicAdd(&sh.h2c[kq], cnt);
                }
                __syncthreads();
                if (rank != 0 && tid < 16 && sh.h2c[tid]) atomicAdd(&L->h2c[tid], sh.h2c[tid]);
                cl.sync();  // S5: the 16 key counts in the leader
                if (tid < 16) sh.xc[tid] = L->h2c[tid];
                __syncthreads();
                const int needk = L->needk;
                int ks = Bk * 16, cnt = 0;
                for (int i = 15; i >= 0; --i) {
                    cnt += (int)sh.xc[i];
                    if (cnt >= needk) {
                        ks = Bk * 16 + i;
                        break;
                    }
                }
                tau = mass_of(__uint_as_float(tp_unkey((uint32_t)ks) << 16), mp);  // tau_k
                Zk = filtered_tiles(tau);
            }
        }
        // ---------------------------------------------------- top-p (R5) on the top-k masses
        uint64_t Zp = Zk;
        if (use_p) {
            // coarse select (leader, all threads): thread t owns bins [4088 - 8t, 4095 - 8t],
            // heaviest first; a block scan of the per-thread masses finds the one thread whose
            // bins cross Theta, which walks them from the heaviest down
            if (rank == 0) {
                unsigned __int128 th = (unsigned __int128)P * Zk + (((unsigned __int128)1 << 32) - 1);
                uint64_t theta = (uint64_t)(th >> 32);
                theta = theta ? theta : 1ull;  // top_p -> 0 keeps the heaviest level (as R5)
                constexpr int PB = TP_H1 / TP_NT;
                const int hb = TP_H1 - 1 - tid * PB;  // this thread's heaviest bin
                uint64_t ls = 0;
#pragma unroll
                for (int i = 0; i < PB; ++i) ls += H1.get(hb - i);
                const uint64_t wincl = warp_incl_scan_u64(ls, lane);
                if (lane == 31) sh.wtot[warp] = wincl;
                __syncthreads();
                uint64_t before = 0;
                for (int w = 0; w < warp; ++w) before += sh.wtot[w];
                const uint64_t incl = before + wincl;  // mass of the bins >= this thread's lowest
                const uint64_t above0 = incl - ls;
                const bool last = tid == TP_NT - 1;
                if ((incl >= theta && above0 < theta) || (last && incl < theta)) {
                    uint64_t above = above0;
                    int B = hb - (PB - 1);
                    for (int i = 0; i < PB; ++i) {
                        const uint64_t h = H1.get(hb - i);
                        if (above + h >= theta) {
                            B = hb - i;
                            break;
                        }
                        above += h;
                    }
                    sh.bsel = B;
                    sh.bz[0] = theta - above;  // mass still needed inside bin B
                    sh.bz[1] = above;
                }
            }
            PH_MARK(4); cl.sync(); PH_MARK(12);  // S6: the leader's coarse select
            if (tid == 0) sh.xB = L->bsel;
            __syncthreads();
            const int B = sh.xB;
            // pass 3: masses of the keys inside bin B (slice -> leader)
            uint32_t c4[4] = {0u, 0u, 0u, 0u};
#ifndef BS_TP_EXP_NOP3  // measurement only: no pass 3
            tp_stream(srow, sbuf, nlt, len, aligned, warp, lane, [&](int, const uint4 v) {
                uint32_t bits[8];
                tp_unpack(v, bits);
#pragma unroll
                for (int i = 0; i < 8; ++i) tp_key_count(c4, tp_key(bits[i]), B);
            });
#endif
#pragma unroll
            for (int kq = 0; kq < 16; ++kq) {
                const uint32_t cnt = tp_warp_count(c4, kq);
                if (lane == 0 && cnt) atomicAdd(&sh.h3c[kq], cnt);
            }
            __syncthreads();
            if (tid < 16) {  // the slice's key masses (count x the key's mass) into its part
                const uint32_t cnt = sh.h3c[tid];
                L->h2part[rank][tid] =
                    cnt ? (uint64_t)cnt * mass_of(__uint_as_float(tp_unkey((uint32_t)(B * 16 + tid)) << 16), mp) : 0ull;
            }
            PH_MARK(5); cl.sync(); PH_MARK(13);  // S7: every slice's key masses in the leader
            if (tid < 16) {  // the cluster's key masses: the 8 parts, loaded together
                unsigned long long pv[TP_CL];
#pragma unroll
                for (int r = 0; r < TP_CL; ++r) pv[r] = L->h2part[r][tid];
                unsigned long long tot = 0;
#pragma unroll
                for (int r = 0; r < TP_CL; ++r) tot += pv[r];
                sh.xh2[tid] = tot;
            }
            if (tid == 16 || tid == 17) sh.xbz[tid - 16] = L->bz[tid - 16];
            __syncthreads();
            // tau = mass(k*) (>= tau_k: Theta <= Z_k); Z' from the histograms unless lower keys
            // share tau (then a filtered pass) — every CTA computes the same values
            const uint64_t need = sh.xbz[0];
            uint64_t above = 0;
            int ks = B * 16;
            for (int i = 15; i >= 0; --i) {
                const uint64_t h = sh.xh2[i];
                if (above + h >= need) {
                    ks = B * 16 + i;
                    break;
                }
                above += h;
            }
            tau = mass_of(__uint_as_float(tp_unkey((uint32_t)ks) << 16), mp);
            Zp = sh.xbz[1] + above + sh.xh2[ks & 15];
            const bool tie_below = ks > 0 && mass_of(__uint_as_float(tp_unkey((uint32_t)ks - 1u) << 16), mp) == tau;
            if (tie_below) Zp = filtered_tiles(tau);
        }
        const uint64_t md_full = (d >= 0) ? mass_of(__uint_as_float((uint32_t)row[d] << 16), mp) : 0ull;
        const uint64_t md = (md_full >= tau) ? md_full : 0ull;  // mass'(d)

        // decision (R7) — every thread of every CTA computes it identically
        bool acc = false;
        if (j < q) acc = uniform_floor(row_draw(a, dsc, PURPOSE_ACCEPT), Zp) < md;
        const int status = acc ? ((a.eos >= 0 && d == a.eos) ? ST_EOS : ST_CONT) : ST_DECIDED;
        if (status == ST_DECIDED) {
            // residual (d excluded) or bonus sample (R8): inverse CDF in ascending id over the
            // slices, then the crossing slice's tiles, then one tile's elements
            if (tiles_tau != tau) filtered_tiles(tau);
            const int excl = (j < q) ? d : -1;
            const uint64_t U = uniform_floor(row_draw(a, dsc, PURPOSE_SAMPLE), Zp - ((j < q) ? md : 0ull));
            const int ex_s = (excl >= 0) ? excl / SL : -1;
            int xs = TP_CL - 1;
            uint64_t us = 0, cum = 0;
            for (int r = 0; r < TP_CL; ++r) {
                const uint64_t ss = tiles_sums[r] - ((r == ex_s) ? md : 0ull);
                if (U < cum + ss) {
                    xs = r;
                    us = U - cum;
                    break;
                }
                cum += ss;
            }
            if (rank == xs && warp == 0) {
                const int per = (nlt + 31) / 32;
                const int i0 = min(nlt, lane * per), i1 = min(nlt, i0 + per);
                const int ex_t = (excl >= 0 && ex_s == rank) ? (excl - e_lo) / 256 : -1;
                uint64_t ls = 0;
                for (int i = i0; i < i1; ++i) ls += sh.tsum[i] - ((i == ex_t) ? md : 0ull);
                const uint64_t incl = warp_incl_scan_u64(ls, lane);
                const unsigned hit = __ballot_sync(0xFFFFFFFFu, us < incl);
                const int Lh = hit ? (__ffs(hit) - 1) : 31;
                int xt = 0;
                uint64_t ut = 0;
                if (lane == Lh) {
                    uint64_t c2 = incl - ls;
                    for (int i = i0; i < i1; ++i) {
                        const uint64_t ts = sh.tsum[i] - ((i == ex_t) ? md : 0ull);
                        if (us < c2 + ts) {
                            xt = i;
                            ut = us - c2;
                            break;
                        }
                        c2 += ts;
                    }
                }
                xt = __shfl_sync(0xFFFFFFFFu, xt, Lh);
                ut = shfl_u64(ut, Lh);
                // rescan tile xt of the slice: lane l owns its 8 elements
                const int e0 = e_lo + xt * 256 + lane * 8;
                const uint4 v = tp_load8(row, e0, min(V, e_lo + len), aligned);
                uint64_t mm[8];
                mass_pair(v.x, mp, mm[0], mm[1]);
                mass_pair(v.y, mp, mm[2], mm[3]);
                mass_pair(v.z, mp, mm[4], mm[5]);
                mass_pair(v.w, mp, mm[6], mm[7]);
                uint64_t s = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (mm[i] < tau || e0 + i == excl || e0 + i >= e_lo + len) mm[i] = 0;
                    s += mm[i];
                }
                const uint64_t inc2 = warp_incl_scan_u64(s, lane);
                const unsigned hit2 = __ballot_sync(0xFFFFFFFFu, ut < inc2);
                const int L2 = hit2 ? (__ffs(hit2) - 1) : 31;
                int tok = -1;
                if (lane == L2) {
                    uint64_t c3 = inc2 - s;
                    for (int i = 0; i < 8; ++i) {
                        c3 += mm[i];
                        if (c3 > ut) {
                            tok = e0 + i;
                            break;
                        }
                    }
                }
                tok = __shfl_sync(0xFFFFFFFFu, tok, L2);
                if (lane == 0) L->cand = tok;
            }
            PH_MARK(6); cl.sync(); PH_MARK(14);  // S8: the sampled token in the leader
        }
        if (rank == 0 && warp == 0) {  // the completion protocol, its finalize in parallel over the warp
            if (lane == 0) sh.stat[STAT_ROWS_VERIFIED] += 1ull;
            int no = 0;
            int32_t tk = -1;
            complete_row_warp(a, sh.stat, dsc.b, j, q, status, status == ST_DECIDED ? sh.cand : -1, Zp,
                              (float)ldexp((double)Z, -a.S), lane, no, tk);
        }
        cl.sync();  // S_end: every CTA is done reading the leader's row state before it is reset
    }
    if (a.stats && tid == 0)
        for (int i = 0; i < STAT_COUNT; ++i)
            if (sh.stat[i]) atomicAdd(a.stats + i, sh.stat[i]);
}
