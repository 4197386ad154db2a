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
// One persistent CTA per row; the row is read from HBM once and re-read from L2.
#pragma once
// (included inside namespace bs)

constexpr int TP_NT = 512;            // threads
constexpr int TP_NW = TP_NT / 32;     // warps
constexpr int TP_H1 = 4096;           // coarse key bins
constexpr int TP_MAXT = 2048;         // 256-element tiles: V <= 524288

struct TopPShared {
    uint32_t h1lo[TP_H1], h1hi[TP_H1];  // coarse-bin masses (Hist64)
    uint32_t hc[TP_H1];       // top-k: positive-mass tokens per coarse bin
    uint32_t h2c[16];         // top-k: positive-mass tokens per key of the crossing bin
    unsigned long long tsum[TP_MAXT];
    uint32_t h2lo[16], h2hi[16];        // masses of the 16 keys of the crossing bin (Hist64)
    unsigned long long stat[STAT_COUNT];
    float wmax[TP_NW];
    uint32_t wbad[TP_NW];
    RowDesc dsc;
    unsigned long long bz[3];  // [0] Theta remaining inside the coarse bin, [1] sum above it, [2] Z
    int32_t bsel;              // coarse bin B
    int32_t bselk, needk;      // top-k: coarse bin of kappa, tokens still needed inside it
};

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

// Stream the row tile by tile (warp w: tiles w, w + TP_NW, ...), TP_U tiles' loads issued
// before any is consumed: one CTA per row, so the passes are bound by how many bytes each warp
// keeps in flight (one 16-byte load per lane at a time was ~1 KB per warp: latency-bound).
#ifndef BS_TP_U
#define BS_TP_U 2
#endif
constexpr int TP_U = BS_TP_U;
template <class F>
__device__ __forceinline__ void tp_stream(const uint16_t* row, int ntile, int V, bool aligned, int warp, int lane,
                                          F&& f) {
    for (int t0 = warp; t0 < ntile; t0 += TP_NW * TP_U) {
        uint4 v[TP_U];
#pragma unroll
        for (int u = 0; u < TP_U; ++u) {
            const int t = t0 + u * TP_NW;
            v[u] = (t < ntile) ? tp_load8(row, t * 256 + lane * 8, V, aligned)
                               : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
        }
#pragma unroll
        for (int u = 0; u < TP_U; ++u) {
            const int t = t0 + u * TP_NW;
            if (t < ntile) f(t, v[u]);  // (warp-uniform)
        }
    }
}

__global__ void __launch_bounds__(TP_NT, 2) verify_topp_kernel(const VerifyArgs a, float top_p, int top_k) {
    extern __shared__ __align__(16) uint8_t tp_smem[];
    TopPShared& sh = *reinterpret_cast<TopPShared*>(tp_smem);
    pdl_wait();  // dependents launch at exit (the cluster kernel plans before its wait)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rows = (int)a.ctl[VCTL_ROWS];
    const int V = a.V;
    const int ntile = (V + 255) / 256;
    const uint64_t P = (uint64_t)llround((double)top_p * 4294967296.0);  // R5 (top_p < 1)
    const bool use_p = top_p < 1.f, use_k = top_k > 0;
    for (int i = tid; i < STAT_COUNT; i += TP_NT) sh.stat[i] = 0ull;

    for (;;) {
        if (tid == 0) sh.dsc = claim_row(a, rows);
        __syncthreads();
        const RowDesc dsc = sh.dsc;
        if (dsc.b < 0) break;
        const uint16_t* row = a.logits + dsc.rowno * a.stride;
        const bool aligned = dsc.aligned != 0;
        const int j = dsc.j, q = dsc.q, d = dsc.d;

        // ---------------------------------------------------- pass 1: max
        uint32_t mx = 0xFF80FF80u;
        tp_stream(row, ntile, V, aligned, warp, lane, [&](int, const uint4 v) {
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
        const Hist64 H1{sh.h1lo, sh.h1hi}, H2{sh.h2lo, sh.h2hi};
        for (int i = tid; i < TP_H1; i += TP_NT) H1.clear(i);
        if (use_k)
            for (int i = tid; i < TP_H1; i += TP_NT) sh.hc[i] = 0u;
        if (tid < 16) {
            H2.clear(tid);
            sh.h2c[tid] = 0u;
        }
        __syncthreads();
        float m = -INFINITY;
        uint32_t bb = 0;
        for (int w = 0; w < TP_NW; ++w) {
            m = fmaxf(m, sh.wmax[w]);
            bb |= sh.wbad[w];
        }
        uint32_t err = 0;
        if (bb) err |= DEV_BAD_LOGIT;
        else if (m == -INFINITY) err |= DEV_ALL_NEGINF;
        else if (!(fabsf(__fmul_rn(m, a.c)) < 16777216.0f)) err |= DEV_RANGE;
        if (err) {  // R0: the row is an error; the rollout stops (no token)
            if (tid == 0) {  // reported at finalize only if Alg. 1 needs this row
                sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                complete_row(a, sh.stat, dsc.b, j, q, ST_ERR, (int)err, 0ull, 0.f);
            }
            __syncthreads();
            continue;
        }
        MassParams mp;
        mp.c = a.c;
        mp.nmc = -__fmul_rn(m, a.c);
        mp.clampv = -(float)(a.S + 2);
        mp.magic = 12582912.0f + (float)a.S;

        // ---------------------------------------------------- pass 2: masses, Z, coarse bins
        tp_stream(row, ntile, V, aligned, warp, lane, [&](int t, const uint4 v) {
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
                    if (use_p) H1.add(kb, mm[i]);
                    if (use_k) atomicAdd(&sh.hc[kb], 1u);
                }
            }
            const uint64_t ws = warp_sum_u51(s);
            if (lane == 0) sh.tsum[t] = ws;
        });
        __syncthreads();
        // pass 4: filtered tile sums (masses >= t); tiles_tau = the t sh.tsum reflects
        uint64_t tiles_tau = 0;  // pass 2's sums keep every mass
        auto filtered_tiles = [&](uint64_t t) {
            __syncthreads();  // earlier readers of sh.tsum are done
            tp_stream(row, ntile, V, aligned, warp, lane, [&](int tt, const uint4 v) {
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
            tiles_tau = t;
        };
        auto tiles_total = [&]() {  // every thread: the sum of sh.tsum
            uint64_t zl = 0;
            for (int t = lane; t < ntile; t += 32) zl += sh.tsum[t];
            return warp_sum_u64(zl);
        };
        const uint64_t Z = tiles_total();  // R4: the unfiltered normaliser
        // ---------------------------------------------------- top-k (R5k): tau_k, Z_k
        uint64_t tau = 0, Zk = Z;
        if (use_k) {
            if (warp == 0) {  // count select over the coarse bins, heaviest first
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
                const int L = hit ? (__ffs(hit) - 1) : 32;
                if (lane == L) {
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
            __syncthreads();
            const int Bk = sh.bselk;
            if (Bk >= 0) {
                // pass 3k: counts of the 16 keys inside bin Bk
                tp_stream(row, ntile, V, aligned, warp, lane, [&](int, const uint4 v) {
                    uint32_t bits[8];
                    tp_unpack(v, bits);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint32_t kk = tp_key(bits[i]);
                        if ((int)(kk >> 4) == Bk && mass_of(__uint_as_float(bits[i] << 16), mp))
                            atomicAdd(&sh.h2c[kk & 15u], 1u);
                    }
                });
                __syncthreads();
                int ks = Bk * 16, cnt = 0;
                for (int i = 15; i >= 0; --i) {
                    cnt += (int)sh.h2c[i];
                    if (cnt >= sh.needk) {
                        ks = Bk * 16 + i;
                        break;
                    }
                }
                tau = mass_of(__uint_as_float(tp_unkey((uint32_t)ks) << 16), mp);  // tau_k
                filtered_tiles(tau);
                Zk = tiles_total();
            }
        }
        // ---------------------------------------------------- top-p (R5) on the top-k masses
        uint64_t Zp = Zk;
        bool tie_below = false;
        if (use_p) {
            // coarse select (warp 0): lane l owns bins [l*128, l*128+128), heaviest first
            if (warp == 0) {
                unsigned __int128 th = (unsigned __int128)P * Zk + (((unsigned __int128)1 << 32) - 1);
                uint64_t theta = (uint64_t)(th >> 32);
                theta = theta ? theta : 1ull;  // top_p -> 0 keeps the heaviest level (as R5)
                const int per = TP_H1 / 32;
                const int lo = (31 - lane) * per;  // lane 0 owns the heaviest bins
                uint64_t ls = 0;
                for (int i = 0; i < per; ++i) ls += H1.get(lo + i);
                const uint64_t incl = warp_incl_scan_u64(ls, lane);  // mass of bins >= lane's lowest
                const unsigned hit = __ballot_sync(0xFFFFFFFFu, incl >= theta);
                const int L = hit ? (__ffs(hit) - 1) : 31;
                if (lane == L) {
                    uint64_t above = incl - ls;
                    int B = lo;
                    for (int i = per - 1; i >= 0; --i) {
                        const uint64_t h = H1.get(lo + i);
                        if (above + h >= theta) {
                            B = lo + i;
                            break;
                        }
                        above += h;
                    }
                    sh.bsel = B;
                    sh.bz[0] = theta - above;  // mass still needed inside bin B
                    sh.bz[1] = above;
                }
            }
            __syncthreads();
            const int B = sh.bsel;
            // pass 3: keys inside bin B
            tp_stream(row, ntile, V, aligned, warp, lane, [&](int, const uint4 v) {
                uint32_t bits[8];
                tp_unpack(v, bits);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t kk = tp_key(bits[i]);
                    if ((int)(kk >> 4) == B) {
                        const uint64_t mi = mass_of(__uint_as_float(bits[i] << 16), mp);
                        if (mi) H2.add(kk & 15u, mi);
                    }
                }
            });
            __syncthreads();
            // tau = mass(k*) (>= tau_k: Theta <= Z_k); Z' from the histograms unless lower keys
            // share tau (then a filtered pass)
            const uint64_t need = sh.bz[0];
            uint64_t above = 0;
            int ks = B * 16;
            for (int i = 15; i >= 0; --i) {
                if (above + H2.get(i) >= need) {
                    ks = B * 16 + i;
                    break;
                }
                above += H2.get(i);
            }
            tau = mass_of(__uint_as_float(tp_unkey((uint32_t)ks) << 16), mp);
            Zp = sh.bz[1] + above + H2.get(ks & 15);
            tie_below = ks > 0 && mass_of(__uint_as_float(tp_unkey((uint32_t)ks - 1u) << 16), mp) == tau;
            if (tie_below) {
                filtered_tiles(tau);
                Zp = tiles_total();
            }
        }
        const uint64_t md_full = (d >= 0) ? mass_of(__uint_as_float((uint32_t)row[d] << 16), mp) : 0ull;
        const uint64_t md = (md_full >= tau) ? md_full : 0ull;  // mass'(d)

        // decision (R7) — every thread computes it identically
        bool acc = false;
        if (j < q) acc = uniform_floor(row_draw(a, dsc, PURPOSE_ACCEPT), Zp) < md;
        const int status = acc ? ((a.eos >= 0 && d == a.eos) ? ST_EOS : ST_CONT) : ST_DECIDED;
        int cand = -1;
        if (status == ST_DECIDED) {
            // residual (d excluded) or bonus sample (R8): inverse CDF in ascending id
            if (tiles_tau != tau) filtered_tiles(tau);
            const int excl = (j < q) ? d : -1;
            const uint64_t U = uniform_floor(row_draw(a, dsc, PURPOSE_SAMPLE), Zp - ((j < q) ? md : 0ull));
            if (warp == 0) {
                const int per = (ntile + 31) / 32;
                const int i0 = min(ntile, lane * per), i1 = min(ntile, i0 + per);
                const int ex_t = (excl >= 0) ? excl / 256 : -1;
                uint64_t ls = 0;
                for (int i = i0; i < i1; ++i) ls += sh.tsum[i] - ((i == ex_t) ? md : 0ull);
                const uint64_t incl = warp_incl_scan_u64(ls, lane);
                const unsigned hit = __ballot_sync(0xFFFFFFFFu, U < incl);
                const int L = hit ? (__ffs(hit) - 1) : 31;
                int xt = 0;
                uint64_t ut = 0;
                if (lane == L) {
                    uint64_t cum = incl - ls;
                    for (int i = i0; i < i1; ++i) {
                        const uint64_t ts = sh.tsum[i] - ((i == ex_t) ? md : 0ull);
                        if (U < cum + ts) {
                            xt = i;
                            ut = U - cum;
                            break;
                        }
                        cum += ts;
                    }
                }
                xt = __shfl_sync(0xFFFFFFFFu, xt, L);
                ut = shfl_u64(ut, L);
                // rescan tile xt: lane l owns its 8 elements
                const int e0 = xt * 256 + lane * 8;
                const uint4 v = tp_load8(row, e0, V, aligned);
                uint64_t mm[8];
                mass_pair(v.x, mp, mm[0], mm[1]);
                mass_pair(v.y, mp, mm[2], mm[3]);
                mass_pair(v.z, mp, mm[4], mm[5]);
                mass_pair(v.w, mp, mm[6], mm[7]);
                uint64_t s = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (mm[i] < tau || e0 + i == excl || e0 + i >= V) mm[i] = 0;
                    s += mm[i];
                }
                const uint64_t inc2 = warp_incl_scan_u64(s, lane);
                const unsigned hit2 = __ballot_sync(0xFFFFFFFFu, ut < inc2);
                const int L2 = hit2 ? (__ffs(hit2) - 1) : 31;
                int tok = -1;
                if (lane == L2) {
                    uint64_t cum = inc2 - s;
                    for (int i = 0; i < 8; ++i) {
                        cum += mm[i];
                        if (cum > ut) {
                            tok = e0 + i;
                            break;
                        }
                    }
                }
                cand = __shfl_sync(0xFFFFFFFFu, tok, L2);
            }
        }
        if (tid == 0) {
            sh.stat[STAT_ROWS_VERIFIED] += 1ull;
            complete_row(a, sh.stat, dsc.b, j, q, status, cand, Zp, (float)ldexp((double)Z, -a.S));
        }
        __syncthreads();
    }
    if (a.stats && tid == 0)
        for (int i = 0; i < STAT_COUNT; ++i)
            if (sh.stat[i]) atomicAdd(a.stats + i, sh.stat[i]);
}
