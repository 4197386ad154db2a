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

constexpr int CK_CL = 8;                  // CTAs per cluster
constexpr int CK_NMW = 6;                 // mass warps: 0..5
constexpr int CK_NXW = 2;                 // max warps: 6..7
constexpr int CK_NCW = CK_NMW + CK_NXW;
constexpr int CK_PROD = CK_NCW;           // producer warp
constexpr int CK_EPI = CK_NCW + 1;        // epilogue warp
constexpr int CK_NT = (CK_NCW + 2) * 32;  // 320 threads
constexpr int CK_NB = 2;                  // slice buffers
constexpr int CK_D = 4;                   // descriptor / exchange ring depth
constexpr int CK_TILE = 512;              // elements per tile (16 per lane)
constexpr int CK_MAXT = 104;              // tiles per slice
constexpr int CK_MAXSL = CK_MAXT * CK_TILE;  // 53248 elements: V <= 425984

struct CkShared {
    uint64_t full[CK_NB], empty[CK_NB];
    uint64_t dfull[CK_D], dempty[CK_D], maxbar[CK_D], sumbar[CK_D], eempty[CK_D];
    RowDesc dq[CK_D];
    uint4 cmax[CK_D][CK_CL];  // per CTA: {slice max bits, bad, greedy index, 0}
    uint4 csum[CK_D][CK_CL];  // per CTA: {slice mass sum lo, hi, mass(d) lo, hi}
    uint4 erec[CK_D];         // mass warps -> epilogue: {m bits, bad, greedy index, 0}
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

// Masses of 16 consecutive logits (two 16-byte vectors), elements >= nvalid or == excl
// zeroed (indices relative to the first element).
__device__ __forceinline__ void ck_mass16(const uint4 v0, const uint4 v1, const MassParams& mp,
                                          int e0, int nvalid, int excl, uint64_t mm[16]) {
    mass8_masked(v0, mp, e0, nvalid, excl, mm);
    mass8_masked(v1, mp, e0 + 8, nvalid, excl, mm + 8);
}

__global__ void __cluster_dims__(CK_CL, 1, 1) __launch_bounds__(CK_NT, 2)
    verify_cluster_kernel(const VerifyArgs a, int SL) {
    pdl_wait();
    pdl_trigger();
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(128) uint8_t ck_smem[];
    CkShared& sh = *reinterpret_cast<CkShared*>(ck_smem);
    uint16_t* bufs = reinterpret_cast<uint16_t*>(ck_smem + ((sizeof(CkShared) + 127) & ~size_t(127)));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rank = (int)cluster.block_rank();
    const int rows = (int)a.ctl[VCTL_ROWS];
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
    cluster.sync();  // every CTA's barriers exist before any remote operation

    if (warp == CK_PROD) {
        // ================================================================ producer
        // The leader claims row i+1 right after issuing row i's copy (one row of lookahead:
        // the claim's dependent loads stay off the compute warps' critical path) and
        // broadcasts each descriptor with 24 lanes (8 CTAs x 3 x 16 bytes).
        const int cid = (int)(blockIdx.x / CK_CL), ncl = (int)(gridDim.x / CK_CL);
        auto broadcast = [&](int r) {
            const int s = r % CK_D;
            // every CTA's epilogue is done with row r-4 (the slot's previous use)
            if (r >= CK_D) mbar_wait_cluster(&sh.dempty[s], ((r / CK_D) - 1) & 1);
            RowDesc nd;
            if (lane == 0) {
                if (r == 0 && cid < rows) nd = a.items[cid];  // first claim: static
                else nd = claim_row(a, rows, ncl);
            }
            uint32_t w[12];
            memcpy(w, &nd, sizeof(w));
#pragma unroll
            for (int x = 0; x < 12; ++x) w[x] = __shfl_sync(0xFFFFFFFFu, w[x], 0);
            if (lane < 3 * CK_CL) {
                const int part = lane % 3;
                uint4 v = make_uint4(w[0], w[1], w[2], w[3]);
                if (part == 1) v = make_uint4(w[4], w[5], w[6], w[7]);
                if (part == 2) v = make_uint4(w[8], w[9], w[10], w[11]);
                st_async_v4(reinterpret_cast<uint4*>(&sh.dq[s]) + part, v, &sh.dfull[s], (uint32_t)(lane / 3));
            }
        };
        if (lane == 0) mbar_arrive_expect_tx(&sh.dfull[0], (uint32_t)sizeof(RowDesc));
        if (rank == 0) broadcast(0);
        for (int i = 0;; ++i) {
            const int s = i % CK_D, bi = i % CK_NB;
            // arm the descriptor slot for row i (its use by row i-4 completed: this warp
            // waited on it); the leader's bytes may already have arrived
            if (i > 0 && lane == 0) mbar_arrive_expect_tx(&sh.dfull[s], (uint32_t)sizeof(RowDesc));
            mbar_wait(&sh.dfull[s], (i / CK_D) & 1);
            const RowDesc dsc = sh.dq[s];
            if (dsc.b < 0) break;
            // the slice buffer is free once the mass warps are done with row i-2
            if (i >= CK_NB) mbar_wait(&sh.empty[bi], ((i / CK_NB) - 1) & 1);
            if (lane == 0) {
                uint16_t* buf = bufs + (size_t)bi * SL;
                const uint16_t* src = a.logits + dsc.rowno * a.stride + e_lo;
                const int nb = dsc.aligned ? (len & ~7) : 0;  // 16-byte multiple
                for (int e = nb; e < len; ++e) buf[e] = src[e];  // ragged end / unaligned row
                if (nb) {
                    fence_proxy_async_smem();
                    mbar_arrive_expect_tx(&sh.full[bi], (uint32_t)nb * 2u);
                    bulk_g2s(buf, src, (uint32_t)nb * 2u, &sh.full[bi], 0ull);
                } else {
                    mbar_arrive(&sh.full[bi]);
                }
            }
            if (rank == 0) broadcast(i + 1);
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
            mbar_wait(&sh.sumbar[s], (i / CK_D) & 1);
            const int b = dsc.b, j = dsc.j, q = dsc.q, d = dsc.d;
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
            const bool lead = rank == 0 && lane == 0;
            if (err) {
                if (lead) {
                    atomicOr(a.dev_err, err);
                    sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                    complete_row(a, sh.stat, b, j, q, ST_DECIDED, -1, 0ull, 0.f);
                }
            } else if (a.T == 0.f) {  // greedy (R1): lowest index attaining m
                const int g = (int)er.z;
                if (lead) {
                    const bool acc = j < q && d == g;
                    const int status = acc ? ((a.eos >= 0 && d == a.eos) ? ST_EOS : ST_CONT) : ST_DECIDED;
                    sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                    complete_row(a, sh.stat, b, j, q, status, g, 1ull, 1.f);
                }
            } else {
                const float norm = (float)ldexp((double)Z, -a.S);
                bool acc = false;
                if (j < q) acc = uniform_floor(row_draw(a, dsc, PURPOSE_ACCEPT), Z) < md;
                const int status = acc ? ((a.eos >= 0 && d == a.eos) ? ST_EOS : ST_CONT) : ST_DECIDED;
                if (status != ST_DECIDED) {
                    if (lead) {
                        sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                        complete_row(a, sh.stat, b, j, q, status, -1, Z, norm);
                    }
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
                        // re-read the tile (L2): lane l owns its 16 consecutive elements
                        const uint16_t* rowp = a.logits + dsc.rowno * a.stride + e_lo;
                        const int e0 = xt * CK_TILE + lane * 16;
                        uint4 v0, v1;
                        if (dsc.aligned && e0 + 16 <= len) {
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
                        if (lane == 0) {
                            sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                            complete_row(a, sh.stat, b, j, q, ST_DECIDED, tok, Z, norm);
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sh.eempty[s]);             // tile sums / sum slot of row i free
                mbar_arrive_remote(&sh.dempty[s], 0u);  // descriptor slot of row i free
            }
        }
    } else if (warp >= CK_NMW) {
        // ================================================================ max warps
        const int xw = warp - CK_NMW;
        for (int i = 0;; ++i) {
            const int s = i % CK_D, bi = i % CK_NB;
            mbar_wait(&sh.dfull[s], (i / CK_D) & 1);
            if (sh.dq[s].b < 0) break;
            // this CTA's epilogue is done with row i-4 (sum slot, tile sums): every peer's
            // row-i publish lands on completed phases of this CTA's rings
            if (i >= CK_D) mbar_wait(&sh.eempty[s], ((i / CK_D) - 1) & 1);
            mbar_wait(&sh.full[bi], (i / CK_NB) & 1);
            const uint16_t* buf = bufs + (size_t)bi * SL;
            uint32_t mx = 0xFF80FF80u;
            for (int t = xw; t < ntile; t += CK_NXW) {
                const int e0 = t * CK_TILE + lane * 16;
                if (t * CK_TILE + CK_TILE <= len) {
                    const uint4 v0 = lds128(buf + e0), v1 = lds128(buf + e0 + 8);
                    mx = hmax2_nan_u32(mx, hmax2_nan_u32(hmax2_nan_u32(v0.x, v0.y), hmax2_nan_u32(v0.z, v0.w)));
                    mx = hmax2_nan_u32(mx, hmax2_nan_u32(hmax2_nan_u32(v1.x, v1.y), hmax2_nan_u32(v1.z, v1.w)));
                } else {
                    for (int x = 0; x < 16; ++x)
                        if (e0 + x < len) mx = hmax2_nan_u32(mx, (uint32_t)buf[e0 + x] | 0xFF800000u);
                }
            }
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
                for (int t = warp; t < ntile; t += CK_NMW) {
                    const int e0 = t * CK_TILE + lane * 16;
                    uint64_t acc;
                    if (t * CK_TILE + CK_TILE <= len) {
                        acc = mass8(lds128(buf + e0), mp) + mass8(lds128(buf + e0 + 8), mp);
                    } else {
                        acc = 0;
                        for (int x = 0; x < 16; ++x)
                            if (e0 + x < len) acc += mass_of(__uint_as_float((uint32_t)buf[e0 + x] << 16), mp);
                    }
                    const uint64_t ts = warp_sum_u51(acc);
                    if (lane == 0) sh.tsum[s][t] = ts;
                    wacc += ts;
                }
            }
            if (lane == 0) sh.wsum[warp] = wacc;
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
            if (lane == 0) mbar_arrive(&sh.empty[bi]);  // slice buffer free
        }
    }
    cluster.sync();  // no CTA exits while a peer may still address its shared memory
    if (a.stats && tid == 0)
        for (int i = 0; i < STAT_COUNT; ++i)
            if (sh.stat[i]) atomicAdd(a.stats + i, sh.stat[i]);
}
