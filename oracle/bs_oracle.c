/*
 * bs_oracle.c — TEST INFRASTRUCTURE ONLY (the parity oracle).
 *
 * A plain, slow, sequential CPU implementation of what the BubbleSpec hot path
 * computes.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this code.  It shares NO code, header, table or
 * constant generator with the CUDA path (paper_2605_08862_b200/csrc); the
 * numeric constants below are restated from DESIGN.md §3 ("reference
 * arithmetic R"), not included from anywhere.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 *   - Eq. 2  (accept with probability p_t(x~))
 *   - Eq. 3  (residual r_t(x) = p_t(x)1[x!=x~]/(1-p_t(x~))) P:208-210
 *   - Alg. 1 (sequential block verification, EOS stop)
 *   - bonus token counted in acceptance length
 *   - p_t after temperature and top-p filtering
 *   - suffix-index draft retrieval, frequency ranked
 * Readings where the paper is silent are DESIGN.md §2 "readings" R0-R8, L1-L6.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared -o libbs_oracle.so bs_oracle.c -lm
 * (-ffp-contract=off so that the only fused multiply-adds are the explicit fmaf()
 * calls that the arithmetic definition R names.)
 *
 * Parity pins: every exported function is pinned by tests/test_oracle_pins.py
 * (Philox KATs, exp2_R closed form, SPEC worked examples, chi-square losslessness,
 * closed-form acceptance, greedy = argmax LCP, brute-force-vs-trie lookup).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_INVALID 1
#define ORC_ERR_DEVICE 7 /* same meaning as BS_ERR_DEVICE: NaN/+inf logits, all -inf row, range */

/* ------------------------------------------------------------------------- */
/* R6: Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).  The paper draws     */
/* "accept with probability p" (Alg.1) without naming a generator;*/
/* reading R6 fixes a counter-based one so the CPU and GPU draw the same u.    */
/* ------------------------------------------------------------------------- */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Counter layout (reading R6): ctr = (position, purpose, uid_lo, uid_hi),
 * key = (seed_lo, seed_hi); r128 = x0*2^96 + x1*2^64 + x2*2^32 + x3.            */
void orc_draw_r128(uint64_t seed, uint64_t uid, uint32_t position, uint32_t purpose,
                   uint32_t out[4]) {
    uint32_t ctr[4] = {position, purpose, (uint32_t)uid, (uint32_t)(uid >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    orc_philox4x32_10(ctr, key, out);
}

/* U = floor(r128 * Zx / 2^128), exactly (reading R6).  The decision
 * U < M  <=>  r128/2^128 < M/Zx, i.e. the real-valued test "u < p" of Eq. 2.   */
uint64_t orc_uniform_floor(const uint32_t r[4], uint64_t Zx) {
    unsigned __int128 rh = ((uint64_t)r[0] << 32) | r[1];
    unsigned __int128 rl = ((uint64_t)r[2] << 32) | r[3];
    unsigned __int128 A = rh * (unsigned __int128)Zx;
    unsigned __int128 B = rl * (unsigned __int128)Zx;
    unsigned __int128 s = A + (B >> 64);
    return (uint64_t)(s >> 64);
}

/* ------------------------------------------------------------------------- */
/* R3: exp2_R.  Degree-5 Horner polynomial for 2^f on [-1/2, 1/2] in fp32 with */
/* explicit fmaf (coefficients frozen in DESIGN.md §3, fitted by               */
/* scripts/fit_exp2_poly.py).                                                  */
/* ------------------------------------------------------------------------- */
static const float ORC_C0 = 0x1.000002p+0f;
static const float ORC_C1 = 0x1.62e428p-1f;
static const float ORC_C2 = 0x1.ebf918p-3f;
static const float ORC_C3 = 0x1.c6b6e4p-5f;
static const float ORC_C4 = 0x1.3d0c54p-7f;
static const float ORC_C5 = 0x1.5c08e6p-10f;

float orc_exp2_poly(float f) {
    float p = ORC_C5;
    p = fmaf(p, f, ORC_C4);
    p = fmaf(p, f, ORC_C3);
    p = fmaf(p, f, ORC_C2);
    p = fmaf(p, f, ORC_C1);
    p = fmaf(p, f, ORC_C0);
    return p;
}

/* R4: S = 62 - ceil(log2 V), rounded down to an even number: every mass is
 * < 2^(S+2), so Z = sum < 2^64.  (Evenness is part of the definition: it lets a
 * fast implementation fold S into the round-half-even constant of R3.)          */
int orc_mass_shift(int V) {
    int lg = 0;
    while (((int64_t)1 << lg) < (int64_t)V) ++lg;
    int S = 62 - lg;
    return S - (S & 1);
}

/* R3+R4: mass(y) = floor(2^S * p(f) * 2^n), n = round-half-even(y), f = y - n.
 * p has 24 significant bits, so p*2^(n+S) is exact in double and floor() is
 * exact.  For y < -(S+2), p*2^(n+S) < 2^(-1) so the mass is 0; that shortcut
 * also covers y = -inf (a -inf logit).                                        */
uint64_t orc_mass_of_y(float y, int S) {
    if (!(y >= -(float)(S + 2))) return 0;
    float n = nearbyintf(y); /* default rounding mode: round half to even */
    float f = y - n;         /* exact: |f| <= 1/2 and y, n share the grid   */
    float p = orc_exp2_poly(f);
    double e = ldexp((double)p, (int)n + S);
    return (uint64_t)floor(e);
}

/* bf16 bits -> fp32 (exact). */
float orc_bf16_to_float(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return f;
}

/* R2: c = fl32(log2(e) / T) computed in double then rounded once.            */
float orc_temp_scale(float T) { return (float)(1.4426950408889634 / (double)T); }

typedef struct {
    uint64_t z;        /* Z' = sum of kept masses (after top-p)       */
    uint64_t z_full;   /* Z before top-p                              */
    float m;           /* row max (R1)                                */
    int32_t greedy;    /* argmax, lowest id (R1); -1 unless T == 0    */
    double norm_fp64;  /* sum_i exp((l_i - m)/T) in double (libm), T>0 */
    float norm_r;      /* Z_full * 2^-S, the R normaliser as fp32       */
} orc_row_stats;

/* ------------------------------------------------------------------------- */
/* Row distribution p_t "after temperature scaling and any top-p filtering"    */
/* (P:202).  Readings R0 (validity), R1 (max / greedy), R2 (scale), R3-R4       */
/* (integer masses), R5 (top-p).  mass[] receives the kept masses mass'_i.    */
/* ------------------------------------------------------------------------- */
/* qsort comparator: masses in descending order (reading R5). */
static int cmp_u64_desc(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x > y ? -1 : (x < y ? 1 : 0);
}

/* R5 on given integer masses (exposed so the SPEC top-p example S:79 can pin it):
 * P = llround(top_p * 2^32); Theta = ceil(P*Z/2^32); G(t) = sum of the masses > t;
 * keep i  <=>  G(mass_i) < Theta   (tie-closed nucleus: the tokens whose strictly
 * heavier tokens have not yet reached top_p).  Zeroes the dropped masses, returns Z'. */
uint64_t orc_top_p_filter(uint64_t* mass, int V, float top_p) {
    uint64_t Z = 0;
    for (int i = 0; i < V; ++i) Z += mass[i];
    if (!(top_p < 1.0f)) return Z;
    uint64_t P = (uint64_t)llround((double)top_p * 4294967296.0);
    unsigned __int128 t = (unsigned __int128)P * Z + (((unsigned __int128)1 << 32) - 1);
    uint64_t theta = (uint64_t)(t >> 32);
    /* sorted copy: G(mass_i) = sum of the sorted values strictly greater than mass_i */
    uint64_t* sorted = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)V);
    memcpy(sorted, mass, sizeof(uint64_t) * (size_t)V);
    qsort(sorted, (size_t)V, sizeof(uint64_t), cmp_u64_desc);
    /* tau = smallest mass value with G(tau) < Theta; keep i <=> mass_i >= tau */
    uint64_t tau = sorted[0], greater = 0;
    for (int r = 0; r < V;) {
        int e = r;
        uint64_t group = 0;
        while (e < V && sorted[e] == sorted[r]) group += sorted[e++];
        if (greater < theta) tau = sorted[r];
        greater += group;
        r = e;
    }
    free(sorted);
    uint64_t zk = 0;
    for (int i = 0; i < V; ++i) {
        if (mass[i] >= tau) zk += mass[i];
        else mass[i] = 0;
    }
    return zk;
}

/* R5k top-k ("any top-p/top-k filtering"; SPEC S:74 applies top-k, then top-p): keep i
 * <=> fewer than top_k tokens have a strictly larger mass, i.e. mass_i >= the top_k-th largest
 * mass (tie-closed like R5: a tie group straddling the k-th place is kept whole).  top_k <= 0
 * or >= V keeps every token.  Zeroes the dropped masses, returns the kept sum.               */
uint64_t orc_top_k_filter(uint64_t* mass, int V, int top_k) {
    uint64_t Z = 0;
    if (top_k <= 0 || top_k >= V) {
        for (int i = 0; i < V; ++i) Z += mass[i];
        return Z;
    }
    uint64_t* sorted = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)V);
    memcpy(sorted, mass, sizeof(uint64_t) * (size_t)V);
    qsort(sorted, (size_t)V, sizeof(uint64_t), cmp_u64_desc);
    uint64_t tau = sorted[top_k - 1];
    free(sorted);
    for (int i = 0; i < V; ++i) {
        if (mass[i] >= tau) Z += mass[i];
        else mass[i] = 0;
    }
    return Z;
}

/* Row distribution with top-k then top-p (R5k, R5); orc_row_dist is top_k = 0. */
int orc_row_dist_k(const uint16_t* row, int V, float T, float top_p, int top_k, uint64_t* mass,
                   orc_row_stats* st);

int orc_row_dist(const uint16_t* row, int V, float T, float top_p, uint64_t* mass,
                 orc_row_stats* st) {
    return orc_row_dist_k(row, V, T, top_p, 0, mass, st);
}

int orc_row_dist_k(const uint16_t* row, int V, float T, float top_p, int top_k, uint64_t* mass,
                   orc_row_stats* st) {
    if (V < 1 || !(T >= 0.0f) || !(top_p > 0.0f) || !(top_p <= 1.0f)) return ORC_ERR_INVALID;
    /* R0 + R1 */
    float m = -INFINITY;
    for (int i = 0; i < V; ++i) {
        uint16_t b = row[i];
        if ((b & 0x7FFFu) > 0x7F80u) return ORC_ERR_DEVICE; /* NaN  */
        if (b == 0x7F80u) return ORC_ERR_DEVICE;             /* +inf */
        float l = orc_bf16_to_float(b);
        if (l > m) m = l;
    }
    if (m == -INFINITY) return ORC_ERR_DEVICE; /* all -inf */
    st->m = m;
    st->greedy = -1;
    if (T == 0.0f) {
        int32_t g = -1;
        for (int i = 0; i < V; ++i)
            if (orc_bf16_to_float(row[i]) == m) { g = i; break; }
        for (int i = 0; i < V; ++i) mass[i] = (i == g) ? 1u : 0u;
        st->greedy = g;
        st->z = st->z_full = 1;
        st->norm_fp64 = 1.0;
        st->norm_r = 1.0f;
        return ORC_OK;
    }
    /* R2 */
    float c = orc_temp_scale(T);
    if (!(c > 0.0f) || isinf(c)) return ORC_ERR_INVALID;
    float mc = m * c;
    if (!(fabsf(mc) < 16777216.0f)) return ORC_ERR_DEVICE;
    int S = orc_mass_shift(V);
    uint64_t Z = 0;
    double nf = 0.0;
    for (int i = 0; i < V; ++i) {
        float l = orc_bf16_to_float(row[i]);
        float y = fmaf(l, c, -mc);
        mass[i] = orc_mass_of_y(y, S);
        Z += mass[i];
        nf += exp(((double)l - (double)m) / (double)T);
    }
    st->z_full = Z;
    st->norm_fp64 = nf;
    st->norm_r = (float)ldexp((double)Z, -S);
    orc_top_k_filter(mass, V, top_k);           /* R5k first ...                 */
    st->z = orc_top_p_filter(mass, V, top_p);   /* ... then R5 on the top-k masses     */
    return ORC_OK;
}

/* R8: inverse CDF in ascending id order on masses with one excluded id
 * (Eq. 3's 1[x != x~]; excl < 0 for none).  Returns min{x : sum_{i<=x, i!=excl} > U}. */
int32_t orc_sample_index(const uint64_t* mass, int V, int32_t excl, uint64_t U) {
    uint64_t c = 0;
    for (int i = 0; i < V; ++i) {
        if (i == excl) continue;
        c += mass[i];
        if (c > U) return i;
    }
    return -1; /* unreachable when U < sum */
}

/* ------------------------------------------------------------------------- */
/* One decoding step of Alg. 1 for one rollout, with the bonus     */
/* token and the empty-draft fallback.              */
/*   rows[j] (j = 0..q) is the target row for generated-token index pos+j,     */
/*   i.e. the distribution after prefix y + d_1..d_j.  Rows are evaluated      */
/*   lazily in Alg. 1 order: row j is touched only if d_1..d_j were accepted.  */
/* Reading R7: accept d_j <=> U(Z'_{j-1}) < mass'_{j-1}(d_j), counter          */
/*   (pos+j-1, ACCEPT=0).  Residual / bonus: counter (pos+s, SAMPLE=1).        */
/* Reading L6: q is clamped to max_len - pos - 1 (the last token is sampled).   */
/* ------------------------------------------------------------------------- */
/* orc_verify_one_r: the step with the uniforms supplied by the caller.  r_acc + 4*j is the
 * r128 of the accept test of d_{j+1} on row j (counter (pos+j, ACCEPT)), r_smp + 4*j the r128
 * of a sample from row j (counter (pos+j, SAMPLE)), j = 0..k.  orc_verify_one fills them from
 * Philox (R6); tests drive every branch of a step with chosen uniforms through this entry
 * (the exact losslessness enumeration of SURVEY c.6 / S:591).                              */
int orc_verify_one_r(const uint16_t* const* rows, int V, float T, float top_p, int32_t top_k, int32_t pos,
                     int32_t max_len, int32_t eos, int32_t finished, const int32_t* draft,
                     int32_t q_in, int32_t k, const uint32_t* r_acc, const uint32_t* r_smp,
                     int32_t* out_tokens, int32_t* out_len, int32_t* out_acc, float* out_norm_r,
                     double* out_norm64, uint64_t* out_z, int32_t* rows_used) {
    *out_len = 0;
    *out_acc = 0;
    *rows_used = 0;
    if (finished || pos >= max_len) return ORC_OK;
    int32_t q = q_in;
    if (q > k) q = k;
    if (q > max_len - pos - 1) q = max_len - pos - 1;
    if (q < 0) q = 0;
    for (int j = 0; j < q; ++j)
        if (draft[j] < 0 || draft[j] >= V) return ORC_ERR_INVALID;
    uint64_t* mass = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)V);
    int n_out = 0;
    int status = ORC_OK;
    for (int j = 0; j <= q; ++j) {
        orc_row_stats st;
        status = orc_row_dist_k(rows[j], V, T, top_p, top_k, mass, &st);
        if (status != ORC_OK) break;
        *rows_used = j + 1;
        if (out_norm_r) out_norm_r[j] = st.norm_r;
        if (out_norm64) out_norm64[j] = st.norm_fp64;
        if (out_z) out_z[j] = st.z;
        if (j < q) {
            int32_t d = draft[j];
            uint64_t U = orc_uniform_floor(r_acc + 4 * j, st.z);
            if (U < mass[d]) { /* accepted (Eq. 2) */
                out_tokens[n_out++] = d;
                *out_acc += 1;
                if (eos >= 0 && d == eos) break; /* Alg. 1: accepted EOS stops */
                continue;
            }
            /* rejected: one recovered token from the residual (Eq. 3) */
            uint64_t Ux = orc_uniform_floor(r_smp + 4 * j, st.z - mass[d]);
            out_tokens[n_out++] = orc_sample_index(mass, V, d, Ux);
            break;
        }
        /* j == q: all q drafts accepted (or q == 0): bonus / plain sample */
        uint64_t Ub = orc_uniform_floor(r_smp + 4 * q, st.z);
        out_tokens[n_out++] = orc_sample_index(mass, V, -1, Ub);
    }
    free(mass);
    *out_len = n_out;
    return status;
}

int orc_verify_one_k(const uint16_t* const* rows, int V, float T, float top_p, int32_t top_k,
                     uint64_t seed, uint64_t uid, int32_t pos, int32_t max_len, int32_t eos,
                     int32_t finished, const int32_t* draft, int32_t q_in, int32_t k,
                     int32_t* out_tokens, int32_t* out_len, int32_t* out_acc, float* out_norm_r,
                     double* out_norm64, uint64_t* out_z, int32_t* rows_used) {
    if (k < 0 || k > 64) return ORC_ERR_INVALID;
    uint32_t r_acc[4 * 65], r_smp[4 * 65];
    for (int j = 0; j <= k; ++j) {
        orc_draw_r128(seed, uid, (uint32_t)(pos + j), 0u, r_acc + 4 * j);
        orc_draw_r128(seed, uid, (uint32_t)(pos + j), 1u, r_smp + 4 * j);
    }
    return orc_verify_one_r(rows, V, T, top_p, top_k, pos, max_len, eos, finished, draft, q_in, k,
                            r_acc, r_smp, out_tokens, out_len, out_acc, out_norm_r, out_norm64,
                            out_z, rows_used);
}

int orc_verify_one(const uint16_t* const* rows, int V, float T, float top_p, uint64_t seed,
                   uint64_t uid, int32_t pos, int32_t max_len, int32_t eos, int32_t finished,
                   const int32_t* draft, int32_t q_in, int32_t k, int32_t* out_tokens,
                   int32_t* out_len, int32_t* out_acc, float* out_norm_r, double* out_norm64,
                   uint64_t* out_z, int32_t* rows_used) {
    return orc_verify_one_k(rows, V, T, top_p, 0, seed, uid, pos, max_len, eos, finished, draft,
                            q_in, k, out_tokens, out_len, out_acc, out_norm_r, out_norm64, out_z,
                            rows_used);
}

/* ------------------------------------------------------------------------- */
/* Draft lookup by brute force (DESIGN.md §2 reading L1-L5; extends S:157-165, */
/* S:183-188; "retrieve a block of candidate tokens conditioned on   */
/* the current prefix", "token node occurrence frequencies").            */
/*  - occurrence of a window w: (sequence, start) with w contiguous inside one */
/*    sequence.  cont(w) = #occurrences followed by at least one token.        */
/*  - anchor m* = max{m in [Lmin, min(M, |y|)] : cont(y[-m:]) >= 1}.           */
/*  - descent: c_j = argmax_c cnt(w c), ties -> lowest id; stop when none.     */
/* The pool is ONE prompt's sequences: tokens[seq_off[s] .. seq_off[s+1]).     */
/* ------------------------------------------------------------------------- */
static int window_at(const int32_t* tokens, int64_t start, int64_t end, const int32_t* w,
                     int wl) {
    if (start + wl > end) return 0;
    for (int t = 0; t < wl; ++t)
        if (tokens[start + t] != w[t]) return 0;
    return 1;
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* Confidence-scored drafts (draft-source variant; reading C1;    */
/* P:405 "selects candidate tokens with higher confidence based on token node occurrence     */
/* frequencies"; Arctic-style min_token_prob): the descent above stops before token c_j when   */
/* its empirical probability cnt(w c_j) / cnt(w) -- cnt(w) = ALL occurrences of the current   */
/* window w, including those that end a sequence -- is below tau = tau_q / 2^32, compared     */
/* exactly in integers: cnt(w c_j) * 2^32 < tau_q * cnt(w).  tau_q = 0 is orc_lookup.          */
int orc_lookup_conf(const int32_t* tokens, const int64_t* seq_off, int32_t n_seqs, const int32_t* ctx,
                    int32_t ctx_len, int32_t M, int32_t Lmin, int32_t K, uint64_t tau_q, int32_t* draft,
                    int32_t* q_out, int32_t* mstar_out);

int orc_lookup(const int32_t* tokens, const int64_t* seq_off, int32_t n_seqs, const int32_t* ctx,
               int32_t ctx_len, int32_t M, int32_t Lmin, int32_t K, int32_t* draft,
               int32_t* q_out, int32_t* mstar_out) {
    return orc_lookup_conf(tokens, seq_off, n_seqs, ctx, ctx_len, M, Lmin, K, 0ull, draft, q_out, mstar_out);
}

int orc_lookup_conf(const int32_t* tokens, const int64_t* seq_off, int32_t n_seqs, const int32_t* ctx,
                    int32_t ctx_len, int32_t M, int32_t Lmin, int32_t K, uint64_t tau_q, int32_t* draft,
                    int32_t* q_out, int32_t* mstar_out) {
    *q_out = 0;
    *mstar_out = 0;
    if (M < 1 || Lmin < 1 || K < 0 || tau_q > (1ull << 32)) return ORC_ERR_INVALID;
    int32_t mmax = ctx_len < M ? ctx_len : M;
    int32_t mstar = 0;
    /* anchor: longest suffix with a continuation */
    for (int32_t m = mmax; m >= Lmin && mstar == 0; --m) {
        const int32_t* w = ctx + ctx_len - m;
        for (int32_t s = 0; s < n_seqs && mstar == 0; ++s) {
            int64_t a = seq_off[s], b = seq_off[s + 1];
            for (int64_t st = a; st + m < b; ++st) /* st+m < b: followed by a token */
                if (window_at(tokens, st, b, w, m)) { mstar = m; break; }
        }
    }
    *mstar_out = mstar;
    if (mstar == 0 || K == 0) return ORC_OK;
    /* occurrences of the anchor (anywhere, including at sequence ends) */
    int64_t total = seq_off[n_seqs] - seq_off[0];
    int64_t* occ_s = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total + 1));
    int64_t* occ_e = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total + 1));
    int32_t* kids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(total + 1));
    int64_t n_occ = 0;
    const int32_t* w = ctx + ctx_len - mstar;
    for (int32_t s = 0; s < n_seqs; ++s) {
        int64_t a = seq_off[s], b = seq_off[s + 1];
        for (int64_t st = a; st < b; ++st)
            if (window_at(tokens, st, b, w, mstar)) { occ_s[n_occ] = st; occ_e[n_occ] = b; ++n_occ; }
    }
    int32_t wl = mstar, q = 0;
    for (int32_t j = 0; j < K; ++j) {
        /* cnt(w c) = number of occurrences of w followed by c */
        int64_t nk = 0;
        for (int64_t o = 0; o < n_occ; ++o)
            if (occ_s[o] + wl < occ_e[o]) kids[nk++] = tokens[occ_s[o] + wl];
        if (nk == 0) break;
        qsort(kids, (size_t)nk, sizeof(int32_t), cmp_i32);
        int32_t best = kids[0];
        int64_t best_n = 0;
        for (int64_t a = 0; a < nk;) {
            int64_t b = a;
            while (b < nk && kids[b] == kids[a]) ++b;
            if (b - a > best_n) { best_n = b - a; best = kids[a]; } /* strict >: lowest id on ties */
            a = b;
        }
        /* reading C1: cnt(w c_j) / cnt(w) below tau stops the draft (n_occ = cnt(w)) */
        if ((uint64_t)best_n * (1ull << 32) < tau_q * (uint64_t)n_occ) break;
        draft[q++] = best;
        int64_t keep = 0;
        for (int64_t o = 0; o < n_occ; ++o)
            if (occ_s[o] + wl < occ_e[o] && tokens[occ_s[o] + wl] == best) {
                occ_s[keep] = occ_s[o]; occ_e[keep] = occ_e[o]; ++keep;
            }
        n_occ = keep;
        ++wl;
    }
    free(occ_s);
    free(occ_e);
    free(kids);
    *q_out = q;
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Draft-source variant: the n-gram linear-scan drafter ("an n-gram-style */
/* scheme that performs pattern matching directly over raw token sequences",    */
/* P:405 "merely performs a linear match of repeated token sequences to return  */
/* the candidate with the longest common prefix"; the paper's Table 7 ablation, */
/* P:389-406).  Reading N1: the anchor is the longest suffix     */
/* y[-n:], n in [n_min, min(n_max, |y|)], that occurs in the prompt's pool       */
/* followed by at least one token; among its occurrences the FIRST in pool order */
/* (sequence index, then position) wins, and the draft is the up to K tokens    */
/* that follow it in its own sequence.  No counting, no index: the scan is      */
/* linear in the pool (the cost the paper attributes to it).            */
/* ------------------------------------------------------------------------- */
int orc_lookup_ngram(const int32_t* tokens, const int64_t* seq_off, int32_t n_seqs,
                     const int32_t* ctx, int32_t ctx_len, int32_t n_min, int32_t n_max, int32_t K,
                     int32_t* draft, int32_t* q_out, int32_t* n_out) {
    *q_out = 0;
    *n_out = 0;
    if (n_min < 1 || n_max < n_min || K < 0) return ORC_ERR_INVALID;
    int32_t top = ctx_len < n_max ? ctx_len : n_max;
    for (int32_t m = top; m >= n_min; --m) {
        const int32_t* w = ctx + ctx_len - m;
        for (int32_t s = 0; s < n_seqs; ++s) {
            int64_t a = seq_off[s], b = seq_off[s + 1];
            for (int64_t st = a; st + m < b; ++st) { /* st+m < b: followed by a token */
                if (!window_at(tokens, st, b, w, m)) continue;
                int32_t q = 0;
                for (int64_t p = st + m; p < b && q < K; ++p) draft[q++] = tokens[p];
                *q_out = q;
                *n_out = m;
                return ORC_OK;
            }
        }
    }
    return ORC_OK;
}
