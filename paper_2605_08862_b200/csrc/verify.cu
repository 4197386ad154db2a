// verify.cu — fused vocab-row verify + resample (Eq. 2, Eq. 3 P:208-210,
// Alg. 1, bonus token P:308) for sm_100a.
//
// Decomposition (kernel K3):
//   * one thread-block CLUSTER of C CTAs per verified logits row; CTA `rank` owns the
//     vocab slice [rank*SL, min(V, (rank+1)*SL)) which a single elected thread stages
//     into shared memory with 1-D bulk async copies (TMA engine, mbarrier completion,
//     L2 evict-first so the draft index stays resident);
//   * pass 1: row max on packed bf16x2 (NaN-propagating) -> cluster max over DSMEM;
//   * pass 2: integer masses of reading R (exact u64 sums, so the decision is
//     independent of reduction order) -> slice sums over DSMEM -> Z, mass(d);
//   * decisions: accept <=> floor(r*Z/2^128) < mass(d) (Philox counter
//     (pos+j, ACCEPT, uid)); if a sample is needed (rejection: residual without d;
//     j == q: bonus) the CTA holding the CDF crossing finds the token by a warp scan
//     over its slice (only the crossing 256-element tile is rescanned per warp step);
//   * the last row of a rollout to finish (atomic counter) applies Alg. 1's first
//     rejection / EOS logic and writes the emitted tokens.
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "ctx.h"
#include "ptx.cuh"

namespace cg = cooperative_groups;

namespace bs {

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
    const int32_t* row_b;
    const int32_t* row_j;
    const int32_t* rb_q;
    const int32_t* rb_base;
    int32_t* done;
    const int32_t* total_rows;
    RowRes* rowres;
    uint32_t* dev_err;
    int32_t* out_tokens;
    int32_t* out_len;
    int32_t* out_acc;
    float* out_norm;
    unsigned long long* out_z;
    unsigned long long* stats;  // bs::STAT_* counters (may be null)
};

struct __align__(16) VShared {
    uint64_t bar;
    // exchanged over DSMEM
    float xmax;
    uint32_t xbad;
    int32_t xfirst;
    int32_t cand;  // written remotely into the leader (rank 0)
    unsigned long long xsum;
    unsigned long long xmassd;
    // CTA-local
    float wmax[32];
    uint32_t wbad[32];
    int32_t wfirst[32];
    unsigned long long wsum[32];
    // broadcast decisions
    float m;
    int32_t ok;
    int32_t greedy;
    int32_t accept;
    int32_t need_sample;
    int32_t excl;
    int32_t cross_rank;
    int32_t wstar;
    unsigned long long z;
    unsigned long long massd;
    unsigned long long ulocal;  // target within this CTA's slice / warp
};

__device__ __forceinline__ uint32_t hmax2_nan_u32(uint32_t a, uint32_t b) {
    __nv_bfloat162 x, y;
    memcpy(&x, &a, 4);
    memcpy(&y, &b, 4);
    __nv_bfloat162 z = __hmax2_nan(x, y);
    uint32_t r;
    memcpy(&r, &z, 4);
    return r;
}

__device__ __forceinline__ uint64_t mass8(const uint4 v, const MassParams& mp) {
    uint64_t s = 0;
    s += mass_of(bf16lo(v.x), mp);
    s += mass_of(bf16hi(v.x), mp);
    s += mass_of(bf16lo(v.y), mp);
    s += mass_of(bf16hi(v.y), mp);
    s += mass_of(bf16lo(v.z), mp);
    s += mass_of(bf16hi(v.z), mp);
    s += mass_of(bf16lo(v.w), mp);
    s += mass_of(bf16hi(v.w), mp);
    return s;
}

__device__ __forceinline__ float bf16_at(const uint16_t* sl, int e) {
    return __uint_as_float((uint32_t)sl[e] << 16);
}

// Finalize rollout b after all its q+1 rows are verified (Alg. 1 lines 10-31).
__device__ void finalize_rollout(const VerifyArgs& a, int b, int q) {
    const int base = a.rb_base[b];
    const int kp1 = a.k + 1;
    int n_out = 0, acc = 0;
    bool ended = false;
    int decided_row = q;
    for (int j = 0; j < q; ++j) {
        const RowRes* rr = a.rowres + base + j;
        const int accept = __ldcg(&rr->accept);
        const int d = a.draft[(int64_t)b * a.k + j];
        if (accept) {
            a.out_tokens[(int64_t)b * kp1 + n_out++] = d;
            ++acc;
            if (a.eos >= 0 && d == a.eos) {  // accepted EOS ends the block, no sample
                ended = true;
                decided_row = j;
                break;
            }
        } else {
            a.out_tokens[(int64_t)b * kp1 + n_out++] = __ldcg(&rr->cand);
            ended = true;
            decided_row = j;
            break;
        }
    }
    if (!ended) a.out_tokens[(int64_t)b * kp1 + n_out++] = __ldcg(&a.rowres[base + q].cand);
    for (int j = n_out; j < kp1; ++j) a.out_tokens[(int64_t)b * kp1 + j] = -1;
    a.out_len[b] = n_out;
    a.out_acc[b] = acc;
    // rows after the decided one were not needed by Alg. 1: report them as 0
    for (int j = decided_row + 1; j <= q; ++j) {
        if (a.out_norm) a.out_norm[(int64_t)b * kp1 + j] = 0.f;
        if (a.out_z) a.out_z[(int64_t)b * kp1 + j] = 0ull;
    }
    if (a.stats) {
        unsigned long long* st = a.stats;
        if (q > 0) {
            atomicAdd(st + STAT_STEPS_SPEC, 1ull);
            atomicAdd(st + STAT_EMIT_SPEC, (unsigned long long)n_out);
            atomicAdd(st + STAT_ACCEPTED, (unsigned long long)acc);
            atomicAdd(st + STAT_PROPOSED, (unsigned long long)q);
            atomicAdd(st + STAT_HIST + min(n_out, STAT_HIST_BINS - 1), 1ull);
        } else {
            atomicAdd(st + STAT_STEPS_PLAIN, 1ull);
            atomicAdd(st + STAT_EMIT_PLAIN, (unsigned long long)n_out);
        }
        atomicAdd(st + STAT_ROWS_VERIFIED, (unsigned long long)(q + 1));
        atomicAdd(st + STAT_ROWS_NEEDED, (unsigned long long)(decided_row + 1));
    }
}

template <int NT>
__global__ void __launch_bounds__(NT) verify_rows_kernel(const VerifyArgs a) {
    constexpr int NW = NT / 32;
    cg::cluster_group cluster = cg::this_cluster();
    const int C = a.C;
    const int rank = (int)cluster.block_rank();
    const int r = blockIdx.x / C;
    if (r >= *a.total_rows) return;  // uniform across the cluster

    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint16_t* sl = reinterpret_cast<uint16_t*>(smem_raw);
    VShared& sh = *reinterpret_cast<VShared*>(smem_raw + (size_t)a.ntiles * 512);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = a.row_b[r], j = a.row_j[r];
    const int q = a.rb_q[b];
    const int slot = a.slots[b];
    const int kp1 = a.k + 1;
    const int64_t rowno = a.row_index ? a.row_index[(int64_t)b * kp1 + j] : (int64_t)b * kp1 + j;
    const uint16_t* row = a.logits + rowno * a.stride;
    const int s0 = rank * a.SL;
    const int s1 = min(a.V, s0 + a.SL);
    const int len = max(0, s1 - s0);
    const uint16_t* src = row + s0;
    const bool aligned = ((reinterpret_cast<uintptr_t>(src) & 15u) == 0);
    const int bulk = aligned ? (len & ~7) : 0;

    // ---- stage the slice: bulk copy (TMA) + plain loads for the ragged part, -inf pad
    if (tid == 0) {
        mbar_init(&sh.bar, 1);
        fence_mbar_init();
    }
    for (int e = bulk + tid; e < a.ntiles * 256; e += NT) sl[e] = (e < len) ? src[e] : (uint16_t)0xFF80u;
    __syncthreads();
    if (tid == 0) {
        if (bulk) {
            const uint64_t pol = policy_evict_first();
            mbar_arrive_expect_tx(&sh.bar, (uint32_t)bulk * 2u);
            constexpr int CH = 8192;  // elements per bulk copy (16 KiB)
            for (int off = 0; off < bulk; off += CH)
                bulk_g2s(sl + off, src + off, (uint32_t)min(CH, bulk - off) * 2u, &sh.bar, pol);
        } else {
            mbar_arrive(&sh.bar);
        }
    }
    const int ntl = (len + 255) >> 8;             // tiles of 256 elements in this slice
    const int tpw = (ntl + NW - 1) / NW;         // tiles per warp (contiguous ranges)
    const int t0 = min(ntl, warp * tpw), t1 = min(ntl, t0 + tpw);
    mbar_wait(&sh.bar, 0);

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
        for (int m = 16; m; m >>= 1) fm = fmaxf(fm, __shfl_xor_sync(0xFFFFFFFFu, fm, m));
        bad = __any_sync(0xFFFFFFFFu, bad) ? 1u : 0u;
        if (lane == 0) {
            sh.wmax[warp] = fm;
            sh.wbad[warp] = bad;
        }
        __syncthreads();
        if (tid == 0) {
            float m = -INFINITY;
            uint32_t bb = 0;
            for (int w = 0; w < NW; ++w) {
                m = fmaxf(m, sh.wmax[w]);
                bb |= sh.wbad[w];
            }
            sh.xmax = m;
            sh.xbad = bb;
        }
    }
    cluster.sync();
    if (tid == 0) {
        float m = -INFINITY;
        uint32_t bb = 0;
        for (int rr = 0; rr < C; ++rr) {
            const VShared* o = cluster.map_shared_rank(&sh, rr);
            m = fmaxf(m, o->xmax);
            bb |= o->xbad;
        }
        int ok = 1;
        uint32_t err = 0;
        if (bb) { ok = 0; err |= DEV_BAD_LOGIT; }
        else if (m == -INFINITY) { ok = 0; err |= DEV_ALL_NEGINF; }
        else if (a.T > 0.f) {
            const float mc = __fmul_rn(m, a.c);
            if (!(fabsf(mc) < 16777216.0f)) { ok = 0; err |= DEV_RANGE; }
        }
        if (err && rank == 0) atomicOr(a.dev_err, err);
        sh.m = m;
        sh.ok = ok;
    }
    __syncthreads();
    const float m = sh.m;
    const bool ok = sh.ok != 0;
    const int d = (j < q) ? a.draft[(int64_t)b * a.k + j] : -1;  // d_{j+1}, tested on row j

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
        if (tid == 0) {
            int f = 0x7FFFFFFF;
            for (int w = 0; w < NW; ++w) f = min(f, sh.wfirst[w]);
            sh.xfirst = (f == 0x7FFFFFFF) ? f : s0 + f;
        }
        cluster.sync();
        if (tid == 0 && rank == 0) {
            int g = 0x7FFFFFFF;
            for (int rr = 0; rr < C; ++rr) g = min(g, cluster.map_shared_rank(&sh, rr)->xfirst);
            sh.greedy = g;
        }
        cluster.sync();
        if (rank == 0 && tid == 0) {
            const int g = ok ? sh.greedy : -1;
            sh.accept = (j < q) ? (d == g) : 0;
            sh.cand = g;
            sh.z = 1ull;
        }
    } else {
        // ---- pass 2: integer masses (R2-R4), exact sums
        MassParams mp;
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
        if (tid == 0) {
            uint64_t s = 0;
            for (int w = 0; w < NW; ++w) s += sh.wsum[w];
            sh.xsum = s;
            sh.xmassd = (ok && d >= s0 && d < s1) ? mass_of(bf16_at(sl, d - s0), mp) : 0ull;
        }
        cluster.sync();
        if (tid == 0) {
            uint64_t sums[8];
            uint64_t Z = 0, md = 0;
            for (int rr = 0; rr < C; ++rr) {
                const VShared* o = cluster.map_shared_rank(&sh, rr);
                sums[rr] = o->xsum;
                Z += o->xsum;
                md += o->xmassd;
            }
            const uint64_t uidv = a.uid[slot];
            const uint32_t position = (uint32_t)(a.pos[slot] + j);
            int accept = 0, need = 1;
            if (ok && j < q) {
                const uint64_t U = uniform_floor(draw(a.seed, uidv, position, PURPOSE_ACCEPT), Z);
                accept = (U < md) ? 1 : 0;
                need = !accept;
            }
            int excl = (j < q) ? d : -1;
            int cross = -1;
            uint64_t ulocal = 0;
            if (ok && need) {
                const uint64_t zx = Z - ((j < q) ? md : 0ull);
                const uint64_t U2 = uniform_floor(draw(a.seed, uidv, position, PURPOSE_SAMPLE), zx);
                uint64_t before = 0;
                for (int rr = 0; rr < C; ++rr) {
                    const int r0 = rr * a.SL, r1 = min(a.V, r0 + a.SL);
                    const uint64_t adj = sums[rr] - ((excl >= r0 && excl < r1) ? md : 0ull);
                    if (U2 < before + adj) {
                        cross = rr;
                        ulocal = U2 - before;
                        break;
                    }
                    before += adj;
                }
            }
            sh.z = Z;
            sh.massd = md;
            sh.accept = accept;
            sh.need_sample = (ok && need) ? 1 : 0;
            sh.excl = excl;
            sh.cross_rank = cross;
            // crossing warp inside this CTA's slice
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
            if (rank == 0) sh.cand = -1;
        }
        __syncthreads();
        // ---- residual / bonus sample: rescan the crossing warp's tiles (R8, ascending id)
        if (sh.need_sample && sh.cross_rank == rank && warp == sh.wstar) {
            const int excl = sh.excl;
            const uint64_t U = sh.ulocal;
            uint64_t run = 0;
            for (int t = t0; t < t1; ++t) {
                const int e0 = t * 256 + lane * 8;
                const uint4 v = lds128(sl + e0);
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
                uint64_t mm[8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    mm[2 * i] = mass_of(bf16lo(w4[i]), mp);
                    mm[2 * i + 1] = mass_of(bf16hi(w4[i]), mp);
                }
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
                        *cluster.map_shared_rank(&sh.cand, 0) = tok;
                    }
                    break;
                }
                run += tot;
            }
        }
    }
    cluster.sync();
    // ---- publish the row result; the last row of the rollout finalizes it
    if (rank == 0 && tid == 0) {
        const uint64_t Z = ok ? sh.z : 0ull;
        const float norm = (a.T == 0.f) ? 1.0f : (float)ldexp((double)Z, -a.S);
        RowRes* rr = a.rowres + r;
        rr->z = Z;
        rr->norm = norm;
        rr->accept = ok ? sh.accept : 0;
        rr->cand = ok ? sh.cand : -1;
        if (a.out_norm) a.out_norm[(int64_t)b * kp1 + j] = ok ? norm : 0.f;
        if (a.out_z) a.out_z[(int64_t)b * kp1 + j] = Z;
        __threadfence();
        const int prev = atomicAdd(a.done + b, 1);
        if (prev == q) {
            __threadfence();
            finalize_rollout(a, b, q);
            a.done[b] = 0;
        }
    }
}

// ---- plan: clamp q per rollout, prefix-sum rows, map row -> (b, j) (one block)
constexpr int PLAN_NT = 1024;
__global__ void __launch_bounds__(PLAN_NT) verify_plan_kernel(
    int n, int k, int V, const int32_t* slots, const int32_t* draft, const int32_t* draft_len,
    const int32_t* pos, const int32_t* max_len, const int32_t* finished, int32_t* rb_q,
    int32_t* rb_base, int32_t* row_b, int32_t* row_j, int32_t* total_rows, int32_t* out_len,
    int32_t* out_acc, int32_t* out_tokens, float* out_norm, unsigned long long* out_z,
    uint32_t* dev_err) {
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
        mine += q + 1;
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
    for (int b = b0; b < b1; ++b) {
        rb_base[b] = excl;
        const int nr = rb_q[b] + 1;
        for (int jj = 0; jj < nr; ++jj) {
            row_b[excl + jj] = b;
            row_j[excl + jj] = jj;
        }
        excl += nr;
    }
    if (tid == 0) *total_rows = total;
}

static int pick_cluster(int V) {
    // slice <= ~76 KB so two CTAs are co-resident per SM (227 KB smem).
    int C = 1;
    while (C < 8 && (int64_t)((V + C - 1) / C) * 2 > 76 * 1024) C <<= 1;
    return C;
}

template <int NT>
static cudaError_t launch_rows(const VerifyArgs& a, int max_rows, cudaStream_t st) {
    const size_t smem = (size_t)a.ntiles * 512 + sizeof(VShared);
    static int configured = -1;  // per device-independent kernel: max dynamic smem set once
    if (configured < (int)smem) {
        cudaError_t e = cudaFuncSetAttribute(verify_rows_kernel<NT>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        configured = 227 * 1024;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(max_rows * a.C), 1, 1);
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
    verify_plan_kernel<<<1, PLAN_NT, 0, st>>>(
        n, k, V, slots, draft, draft_len, ctx->pos.p, ctx->max_len.p, ctx->finished.p, ctx->rb_q.p,
        ctx->rb_base.p, ctx->row_b.p, ctx->row_j.p, ctx->total_rows.p, out_len, out_acc,
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
    a.row_b = ctx->row_b.p;
    a.row_j = ctx->row_j.p;
    a.rb_q = ctx->rb_q.p;
    a.rb_base = ctx->rb_base.p;
    a.done = ctx->done_ctr.p;
    a.total_rows = ctx->total_rows.p;
    a.rowres = ctx->rowres.p;
    a.dev_err = ctx->dev_err.p;
    a.out_tokens = out_tokens;
    a.out_len = out_len;
    a.out_acc = out_acc;
    a.out_norm = out_norm;
    a.out_z = out_z;
    a.stats = ctx->stats.p;
    const int max_rows = n * (k + 1);
    if (a.SL >= 8192) return launch_rows<512>(a, max_rows, st);
    return launch_rows<128>(a, max_rows, st);
}

}  // namespace bs
