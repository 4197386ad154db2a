// verify_split.cuh — the same verify + resample (reading R, Alg. 1) with each logits row
// split across an 8-CTA thread-block cluster, for steps with few live rows (the long tail
// of a rollout batch, where one CTA per row leaves the GPU idle and the step's
// latency is one row's).  Included by verify.cu inside namespace bs.
//
// Per row (one cluster, persistent over the row queue):
//   * CTA r bulk-copies its slice [r*SL, (r+1)*SL) of the row into shared memory (4 pieces,
//     one mbarrier each, so the max starts on the first piece while the rest lands);
//   * pass 1: slice max (greedy: and its lowest index); the 8 slice results are exchanged
//     over DSMEM (each CTA stores its result into every CTA) and one cluster barrier;
//   * pass 2: masses from shared memory (no second read of the row), 256-element tile sums
//     kept locally, the slice sum exchanged over DSMEM, cluster barrier;
//   * every CTA computes Z and the decision identically; the sample's crossing slice is
//     found from the slice sums and that CTA rescans one tile from its shared memory.
// Rows are claimed from the same queue (j-major, skipping decided rows) and completed with
// the same out-of-order protocol as verify_rows_kernel.
#pragma once
// (included inside namespace bs)

constexpr int SP_CL = 8;        // CTAs per cluster: one row per cluster
constexpr int SP_NT = 256;      // threads per CTA
constexpr int SP_NW = SP_NT / 32;
constexpr int SP_NP = 4;        // slice pieces (mbarriers)
constexpr int SP_MAXT = 256;    // tiles per slice: V <= 8 * 256 * 256

struct SplitShared {
    uint64_t bar[SP_NP];
    RowDesc dsc;
    float cmax[SP_CL];                 // per-CTA slice results (written remotely)
    uint32_t cbad[SP_CL];
    int32_t cidx[SP_CL];
    unsigned long long csum[SP_CL];
    unsigned long long cmd[SP_CL];     // mass(d) from the CTA whose slice holds d, else 0
    float wmax[SP_NW];
    uint32_t wbad[SP_NW];
    int32_t widx[SP_NW];
    unsigned long long wsum[SP_NW];
    unsigned long long tsum[SP_MAXT];
    unsigned long long stat[STAT_COUNT];
    int32_t dec[4];                    // [0] status, [1] crossing CTA, [2] excl
    unsigned long long decz[3];        // [0] Z, [1] U local to the crossing slice, [2] mass(d)
};

__global__ void __cluster_dims__(SP_CL, 1, 1) __launch_bounds__(SP_NT, 2)
    verify_split_kernel(const VerifyArgs a, int SL) {
    pdl_wait();  // dependents launch at exit (the cluster kernel plans before its wait)
    if (a.ctl[VCTL_MODE] != 1) return;  // the plan kernel chose the one-CTA-per-row path
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(128) uint8_t sp_smem[];
    SplitShared& sh = *reinterpret_cast<SplitShared*>(sp_smem);
    uint16_t* slice = reinterpret_cast<uint16_t*>(sp_smem + ((sizeof(SplitShared) + 127) & ~size_t(127)));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rank = (int)cluster.block_rank();
    const int rows = (int)a.ctl[VCTL_ROWS];
    const int cid = (int)(blockIdx.x / SP_CL), ncl = (int)(gridDim.x / SP_CL);
    const int V = a.V;
    const int e_lo = rank * SL;
    const int len = max(0, min(SL, V - e_lo));
    const int ntile = (len + 255) / 256;
    const int tpp = (SL / 256 + SP_NP - 1) / SP_NP;  // tiles per piece
    if (tid == 0) {
        for (int i = 0; i < SP_NP; ++i) mbar_init(&sh.bar[i], 1);
        fence_mbar_init();
    }
    for (int i = tid; i < STAT_COUNT; i += SP_NT) sh.stat[i] = 0ull;
    MassParams mp;
    mp.c = a.c;
    mp.clampv = -(float)(a.S + 2);
    mp.magic = 12582912.0f + (float)a.S;
    __syncthreads();

    int next = cid;  // (leader) next table row of this cluster
    for (uint32_t it = 0;; ++it) {
        if (rank == 0 && tid == 0) {  // static claim: table rows cid, cid + ncl, ...
            RowDesc nd;
            nd.b = -1;
            for (; next < rows; next += ncl) {
                const RowDesc cand = a.items[next];
                if (cand.j > ld_volatile_i32(a.roll_first + cand.b)) continue;  // decided below
                nd = cand;
                next += ncl;
                break;
            }
            for (int r = 0; r < SP_CL; ++r) *cluster.map_shared_rank(&sh.dsc, r) = nd;
        }
        cluster.sync();
        const RowDesc dsc = sh.dsc;
        if (dsc.b < 0) break;
        const uint16_t* row = a.logits + dsc.rowno * a.stride;
        const int j = dsc.j, q = dsc.q, d = dsc.d;

        // ---- slice -> shared memory
        if (tid == 0) {
            const bool bulk_ok = dsc.aligned != 0;
            for (int p = 0; p < SP_NP; ++p) {
                const int p0 = min(len, p * tpp * 256), p1 = min(len, (p + 1) * tpp * 256);
                const int nb = bulk_ok ? ((p1 - p0) & ~7) : 0;  // 16-byte multiple
                for (int e = p0 + nb; e < p1; ++e) slice[e] = row[e_lo + e];  // ragged end
                if (nb) {
                    fence_proxy_async_smem();
                    mbar_arrive_expect_tx(&sh.bar[p], (uint32_t)nb * 2u);
                    bulk_g2s(slice + p0, row + e_lo + p0, (uint32_t)nb * 2u, &sh.bar[p], 0ull);
                } else {
                    mbar_arrive(&sh.bar[p]);
                }
            }
        }
        const uint32_t ph = it & 1u;

        // ---- pass 1: slice max
        uint32_t mx = 0xFF80FF80u;
        for (int t = warp; t < ntile; t += SP_NW) {
            mbar_wait(&sh.bar[t / tpp], ph);
            const int e0 = t * 256 + lane * 8;
            if (t * 256 + 256 <= len) {
                const uint4 v = lds128(slice + e0);
                mx = hmax2_nan_u32(mx, v.x);
                mx = hmax2_nan_u32(mx, v.y);
                mx = hmax2_nan_u32(mx, v.z);
                mx = hmax2_nan_u32(mx, v.w);
            } else {
                for (int i = 0; i < 8; ++i)
                    if (e0 + i < len) mx = hmax2_nan_u32(mx, (uint32_t)slice[e0 + i] | 0xFF800000u);
            }
        }
        for (int p = warp; p < SP_NP; p += SP_NW) mbar_wait(&sh.bar[p], ph);  // every phase consumed
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
        float sm = -INFINITY;
        uint32_t sbad = 0;
        for (int w = 0; w < SP_NW; ++w) {
            sm = fmaxf(sm, sh.wmax[w]);
            sbad |= sh.wbad[w];
        }
        int sidx = 0x7FFFFFFF;
        if (a.T == 0.f && sm > -INFINITY) {  // greedy: lowest index attaining the slice max
            int fi = 0x7FFFFFFF;
            for (int t = warp; t < ntile && fi == 0x7FFFFFFF; t += SP_NW) {
                const int e0 = t * 256 + lane * 8;
                int li = 0x7FFFFFFF;
                for (int i = 7; i >= 0; --i)
                    if (e0 + i < len && __uint_as_float((uint32_t)slice[e0 + i] << 16) == sm) li = e0 + i;
#pragma unroll
                for (int mm = 16; mm; mm >>= 1) li = min(li, __shfl_xor_sync(0xFFFFFFFFu, li, mm));
                fi = li;  // tiles of a warp ascend: the first hit is the warp's lowest
            }
            if (lane == 0) sh.widx[warp] = fi;
            __syncthreads();
            for (int w = 0; w < SP_NW; ++w) sidx = min(sidx, sh.widx[w]);
            if (sidx != 0x7FFFFFFF) sidx += e_lo;
        }
        if (tid == 0) {
            for (int r = 0; r < SP_CL; ++r) {
                *cluster.map_shared_rank(&sh.cmax[rank], r) = sm;
                *cluster.map_shared_rank(&sh.cbad[rank], r) = sbad;
                *cluster.map_shared_rank(&sh.cidx[rank], r) = sidx;
            }
        }
        cluster.sync();
        float m = -INFINITY;
        uint32_t bb = 0;
        for (int r = 0; r < SP_CL; ++r) {
            m = fmaxf(m, sh.cmax[r]);
            bb |= sh.cbad[r];
        }
        uint32_t err = 0;
        if (bb) err |= DEV_BAD_LOGIT;
        else if (m == -INFINITY) err |= DEV_ALL_NEGINF;
        else if (a.T > 0.f && !(fabsf(__fmul_rn(m, a.c)) < 16777216.0f)) err |= DEV_RANGE;
        if (err) {
            if (rank == 0 && tid == 0) {  // reported at finalize only if Alg. 1 needs this row
                sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                complete_row(a, sh.stat, dsc.b, j, q, ST_ERR, (int)err, 0ull, 0.f);
            }
            continue;
        }
        if (a.T == 0.f) {  // greedy (R1)
            int g = 0x7FFFFFFF;
            for (int r = 0; r < SP_CL; ++r)
                if (sh.cmax[r] == m) g = min(g, sh.cidx[r]);
            if (rank == 0 && tid == 0) {
                const bool acc = j < q && d == g;
                const int status = acc ? ((a.eos >= 0 && d == a.eos) ? ST_EOS : ST_CONT) : ST_DECIDED;
                sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                complete_row(a, sh.stat, dsc.b, j, q, status, g, 1ull, 1.f);
            }
            continue;
        }
        mp.nmc = -__fmul_rn(m, a.c);

        // ---- pass 2: masses from shared memory, tile sums
        uint64_t wacc = 0;
        for (int t = warp; t < ntile; t += SP_NW) {
            const int e0 = t * 256 + lane * 8;
            uint64_t s = 0;
            if (t * 256 + 256 <= len) {
                s = mass8(lds128(slice + e0), mp);
            } else {
                for (int i = 0; i < 8; ++i)
                    if (e0 + i < len) s += mass_of(__uint_as_float((uint32_t)slice[e0 + i] << 16), mp);
            }
            const uint64_t ts = warp_sum_u51(s);
            if (lane == 0) sh.tsum[t] = ts;
            wacc += ts;
        }
        if (lane == 0) sh.wsum[warp] = wacc;
        __syncthreads();
        if (tid == 0) {
            uint64_t cs = 0;
            for (int w = 0; w < SP_NW; ++w) cs += sh.wsum[w];
            const int dl = d - e_lo;
            const uint64_t mdl = (d >= 0 && dl >= 0 && dl < len)
                                     ? mass_of(__uint_as_float((uint32_t)slice[dl] << 16), mp)
                                     : 0ull;
            for (int r = 0; r < SP_CL; ++r) {
                *cluster.map_shared_rank(&sh.csum[rank], r) = cs;
                *cluster.map_shared_rank(&sh.cmd[rank], r) = mdl;
            }
        }
        cluster.sync();

        // ---- decision (R7) and the sample's crossing slice (R8), identical in every CTA
        if (tid == 0) {
            uint64_t Z = 0, md = 0;
            for (int r = 0; r < SP_CL; ++r) {
                Z += sh.csum[r];
                md += sh.cmd[r];
            }
            bool acc = false;
            if (j < q) acc = uniform_floor(row_draw(a, dsc, PURPOSE_ACCEPT), Z) < md;
            const int status = acc ? ((a.eos >= 0 && d == a.eos) ? ST_EOS : ST_CONT) : ST_DECIDED;
            int rc = -1;
            uint64_t ul = 0;
            const int excl = (j < q) ? d : -1;
            if (status == ST_DECIDED) {
                const uint64_t U = uniform_floor(row_draw(a, dsc, PURPOSE_SAMPLE), Z - ((j < q) ? md : 0ull));
                const int exr = (excl >= 0) ? excl / SL : -1;
                uint64_t cum = 0;
                for (int r = 0; r < SP_CL; ++r) {
                    const uint64_t cs = sh.csum[r] - ((r == exr) ? md : 0ull);
                    if (U < cum + cs) {
                        rc = r;
                        ul = U - cum;
                        break;
                    }
                    cum += cs;
                }
            }
            sh.dec[0] = status;
            sh.dec[1] = rc;
            sh.dec[2] = excl;
            sh.decz[0] = Z;
            sh.decz[1] = ul;
            sh.decz[2] = md;
            if (status != ST_DECIDED && rank == 0) {  // accepted: no sample
                sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                complete_row(a, sh.stat, dsc.b, j, q, status, -1, Z,
                             (float)ldexp((double)Z, -a.S));
            }
        }
        __syncthreads();
        if (sh.dec[0] == ST_DECIDED && sh.dec[1] == rank && warp == 0) {
            // the crossing tile of this slice (excluded token's mass taken off its tile)
            const int excl_l = sh.dec[2] - e_lo;  // slice-relative (may be out of range)
            const uint64_t md = sh.decz[2], U = sh.decz[1];
            const int ex_t = (excl_l >= 0 && excl_l < len) ? excl_l / 256 : -1;
            const int per = (ntile + 31) / 32;
            const int i0 = min(ntile, lane * per), i1 = min(ntile, i0 + per);
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
            const int e0 = xt * 256 + lane * 8;
            uint64_t mm[8];
            const uint4 v = (xt * 256 + 256 <= len)
                                ? lds128(slice + e0)
                                : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
            if (xt * 256 + 256 <= len) {
                mass8_masked(v, mp, e0, len, excl_l, mm);
            } else {
                for (int i = 0; i < 8; ++i)
                    mm[i] = (e0 + i < len && e0 + i != excl_l)
                                ? mass_of(__uint_as_float((uint32_t)slice[e0 + i] << 16), mp)
                                : 0ull;
            }
            uint64_t s = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) s += mm[i];
            const uint64_t inc2 = warp_incl_scan_u64(s, lane);
            const unsigned hit2 = __ballot_sync(0xFFFFFFFFu, ut < inc2);
            const int L2 = hit2 ? (__ffs(hit2) - 1) : 31;
            int tok = -1;
            if (lane == L2) {
                uint64_t cum = inc2 - s;
                for (int i = 0; i < 8; ++i) {
                    cum += mm[i];
                    if (cum > ut) {
                        tok = e_lo + e0 + i;
                        break;
                    }
                }
            }
            tok = __shfl_sync(0xFFFFFFFFu, tok, L2);
            if (lane == 0) {
                const uint64_t Z = sh.decz[0];
                sh.stat[STAT_ROWS_VERIFIED] += 1ull;
                complete_row(a, sh.stat, dsc.b, j, q, ST_DECIDED, tok, Z, (float)ldexp((double)Z, -a.S));
            }
        }
    }
    __syncthreads();
    if (a.stats && tid == 0)
        for (int i = 0; i < STAT_COUNT; ++i)
            if (sh.stat[i]) atomicAdd(a.stats + i, sh.stat[i]);
}
