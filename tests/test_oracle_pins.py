"""Pins for the CPU oracle: each check compares the oracle with something the paper or
the mathematics fixes — never with the CUDA path and never by retyping the oracle's own
formula.  (Runs on CPU: ``-m "not gpu"``.)
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from workloads import bf16_bits_to_f32, f32_to_bf16_bits

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
LOG2E = 1.4426950408889634


def bf16_row(vals):
    return f32_to_bf16_bits(np.asarray(vals, dtype=np.float32))


# ------------------------------------------------------------------ Philox (R6)
def test_philox_known_answer_vectors(orc):
    """Random123 KAT vectors (tests/golden/philox4x32_10_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        assert orc.philox4x32_10(w[0:4], w[4:6]) == w[6:10]
        n += 1
    assert n == 3


def test_uniform_floor_special_cases(orc):
    """U = floor(r Z / 2^128): SPEC S:88 (u = 0.25 -> first half, 0.75 -> second half)."""
    assert orc.uniform_floor([0x40000000, 0, 0, 0], 2) == 0          # u = 1/4
    assert orc.uniform_floor([0xC0000000, 0, 0, 0], 2) == 1          # u = 3/4
    assert orc.uniform_floor([0xFFFFFFFF] * 4, 1) == 0               # U < Z always
    assert orc.uniform_floor([0xFFFFFFFF] * 4, 2**64 - 1) == 2**64 - 2
    assert orc.uniform_floor([0, 0, 0, 0], 2**64 - 1) == 0


def test_uniform_floor_is_exact_floor(orc):
    """The 64-bit-halves evaluation equals the plain bigint definition floor(r*Z/2^128)."""
    rng = np.random.default_rng(5)
    for _ in range(2000):
        r = [int(x) for x in rng.integers(0, 2**32, size=4, dtype=np.uint64)]
        Z = int(rng.integers(1, 2**63, dtype=np.uint64)) * int(rng.integers(1, 3))
        Z = min(Z, 2**64 - 1)
        r128 = (r[0] << 96) | (r[1] << 64) | (r[2] << 32) | r[3]
        assert orc.uniform_floor(r, Z) == (r128 * Z) >> 128


def test_draw_counter_layout(orc):
    """ctr = (position, purpose, uid_lo, uid_hi), key = (seed_lo, seed_hi) (reading R6)."""
    seed, uid = 0x1122334455667788, 0x99AABBCCDDEEFF00
    got = orc.draw_r128(seed, uid, 7, 1)
    want = orc.philox4x32_10([7, 1, uid & 0xFFFFFFFF, uid >> 32],
                             [seed & 0xFFFFFFFF, seed >> 32])
    assert got == want


# ------------------------------------------------------------------ exp2_R (R3/R4)
def test_exp2_poly_relative_error_closed_form(orc):
    """|p(f)/2^f - 1| <= 2.5e-7 on a dense fp32 grid of [-1/2, 1/2] (closed form 2^f)."""
    fs = np.float32(np.linspace(-0.5, 0.5, 20001))
    worst = max(abs(orc.exp2_poly(float(f)) / 2.0 ** float(f) - 1.0) for f in fs)
    assert worst <= 2.5e-7, worst


def test_mass_shift_values(orc):
    """R4: S = 62 - ceil(log2 V), rounded down to even; Z < 2^64 for any row."""
    assert orc.mass_shift(151936) == 44
    assert orc.mass_shift(1024) == 52
    assert orc.mass_shift(1025) == 50
    assert orc.mass_shift(4) == 60
    assert orc.mass_shift(2) == 60
    assert orc.mass_shift(1) == 62


def test_mass_of_y_against_exp2(orc):
    """mass(y)/2^S = 2^y within the polynomial bound plus one fixed-point ulp; special cases."""
    S = 44
    rng = np.random.default_rng(1)
    ys = np.concatenate([np.float32(rng.uniform(-47, 0.5, 3000)),
                         np.float32([0.0, -0.5, 0.5, -1.5, -2.5, -44.0, -45.9])])
    for y in ys:
        m = orc.mass_of_y(float(y), S)
        exact = 2.0 ** float(y) * 2.0 ** S
        assert abs(m - exact) <= 2.6e-7 * exact + 1.0, (y, m, exact)
    # p(0) = C0 = 1 + 2^-23 exactly, so mass(0) = 2^S + 2^(S-23)
    assert orc.mass_of_y(0.0, S) == 2**S + 2**(S - 23)
    assert orc.mass_of_y(-1.0, S) == 2**(S - 1) + 2**(S - 24)
    assert orc.mass_of_y(float("-inf"), S) == 0
    assert orc.mass_of_y(-(S + 2.5), S) == 0
    assert orc.mass_of_y(-(S + 1.0), S) == 0  # 2^-(S+1) * 2^S = 1/2 -> floor 0


def test_temp_scale(orc):
    """R2: c = fl32(log2 e / T); T = 1 -> 0x3FB8AA3B."""
    assert np.float32(orc.temp_scale(1.0)).view(np.uint32) == 0x3FB8AA3B
    assert orc.temp_scale(float(np.float32(LOG2E))) == 1.0


# ------------------------------------------------------------------ row distribution
def test_row_masses_exact_powers_of_two(orc):
    """With c = 1 (T = fl32(log2 e)), logits {0,-1,-2,-3} give masses C0 * 2^(S-j)."""
    T = float(np.float32(LOG2E))
    V = 4
    d = orc.row_dist(bf16_row([0.0, -1.0, -2.0, -3.0]), T)
    S = orc.mass_shift(V)
    c0 = 2**S + 2**(S - 23)
    assert [int(x) for x in d.mass] == [c0 >> j for j in range(4)]
    assert d.z == sum(c0 >> j for j in range(4))


def test_row_normaliser_vs_fp64(orc):
    """Z * 2^-S equals sum_i exp((l_i - m)/T) (libm, fp64) within 1e-6 relative — the
    north_star's 1e-5 normaliser bar with margin."""
    rng = np.random.default_rng(2)
    for V, T in [(1024, 1.0), (1000, 0.7), (4096, 1.3), (151936, 1.0)]:
        row = bf16_row(rng.normal(0, 2.5, V))
        d = orc.row_dist(row, T)
        l = bf16_bits_to_f32(row).astype(np.float64)
        ref = float(np.sum(np.exp((l - l.max()) / float(np.float32(T)))))
        S = orc.mass_shift(V)
        assert abs(d.z_full / 2.0**S / ref - 1) < 1e-6
        assert abs(d.norm_r / ref - 1) < 1e-6
        assert abs(d.norm_fp64 / ref - 1) < 1e-12


def test_z_fits_64_bits_worst_case(orc):
    """R4 bound: a row of V equal maximal logits has Z = V * mass(y~0) < 2^64."""
    for V in [1, 2, 3, 1000, 1024, 1025, 4096]:
        d = orc.row_dist(bf16_row([7.0] * V), 1.0)
        assert 0 < d.z < 2**64 and d.z == V * int(d.mass[0])


def test_uniform_row_masses_equal(orc):
    for v in [0.0, 3.5, -17.25]:
        d = orc.row_dist(bf16_row([v] * 37), 0.9)
        assert len(set(int(x) for x in d.mass)) == 1
        assert d.z == 37 * int(d.mass[0])


def test_greedy_is_argmax_lowest_id(orc):
    """R1 / S:74: T = 0 is the degenerate distribution on the argmax, ties -> lowest id."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        row = bf16_row(np.round(rng.normal(0, 2, 300)))  # many ties
        d = orc.row_dist(row, 0.0)
        g = int(np.argmax(bf16_bits_to_f32(row)))  # numpy: first occurrence
        assert d.greedy == g and d.z == 1 and int(d.mass[g]) == 1 and int(d.mass.sum()) == 1


def test_invalid_rows(orc):
    """R0: NaN or +inf -> error; all -inf -> error; -inf entries get mass 0."""
    with pytest.raises(orc.OracleError):
        orc.row_dist(np.array([0x3F80, 0x7FC0], dtype=np.uint16), 1.0)
    with pytest.raises(orc.OracleError):
        orc.row_dist(np.array([0x3F80, 0x7F80], dtype=np.uint16), 1.0)
    with pytest.raises(orc.OracleError):
        orc.row_dist(np.array([0xFF80, 0xFF80], dtype=np.uint16), 1.0)
    d = orc.row_dist(np.array([0x3F80, 0xFF80], dtype=np.uint16), 1.0)
    assert int(d.mass[1]) == 0 and int(d.mass[0]) > 0


# ------------------------------------------------------------------ top-p (R5)
def test_top_p_spec_example(orc):
    """(0.5,0.3,0.2), top_p 0.7 -> kept {0,1}, renormalised (0.625, 0.375, 0)."""
    for k in [0, 10, 40]:
        m, z = orc.top_p_filter([5 << k, 3 << k, 2 << k], 0.7)
        assert [Fraction(int(x), z) for x in m] == [Fraction(5, 8), Fraction(3, 8), 0]
    m, z = orc.top_p_filter([5, 3, 2], 0.5)      # cumulative 0.5 >= 0.5 after {0}
    assert list(m) == [5, 0, 0] and z == 5
    m, z = orc.top_p_filter([2, 3, 5], 0.75)     # order is by mass, not by id
    assert list(m) == [0, 3, 5] and z == 8
    m, z = orc.top_p_filter([3, 3, 3, 1], 0.5)   # a tie straddling top_p is kept whole
    assert list(m) == [3, 3, 3, 0] and z == 9
    m, z = orc.top_p_filter([3, 1, 1, 1, 1, 1], 0.375)  # {3} reaches 3/8 exactly: tie dropped
    assert list(m) == [3, 0, 0, 0, 0, 0] and z == 3
    m, z = orc.top_p_filter([3, 1, 1, 1, 1, 1], 0.376)  # ... just above: the whole tie joins
    assert list(m) == [3, 1, 1, 1, 1, 1] and z == 8
    m, z = orc.top_p_filter([1, 7], 1.0)         # identity
    assert list(m) == [1, 7] and z == 8
    m, z = orc.top_p_filter([1, 7], 1e-9)        # never empties the support
    assert list(m) == [0, 7]


def test_top_p_nucleus_properties(orc):
    """The kept set is the smallest tie-closed set of heaviest tokens whose mass reaches
    top_p * Z (checked with exact fractions, by brute force over the distinct mass levels),
    and it grows monotonically with top_p.  (SPEC S:97 also claims idempotence; with
    renormalisation that is false in general, e.g. (0.6, 0.3, 0.1) at top_p 0.65 ->
    {0.6, 0.3} -> {0.6} — DESIGN.md reading R5.)"""
    rng = np.random.default_rng(4)
    for trial in range(300):
        hi = 1000 if trial % 2 else 6          # small value range -> many ties
        m0 = rng.integers(0, hi, 20).astype(np.uint64)
        m0[0] += 1
        Z = int(m0.sum())
        prev_kept = set()
        for p in sorted(float(np.float32(x)) for x in rng.uniform(0.01, 1.0, 4)):
            m1, z1 = orc.top_p_filter(m0, p)
            kept = {i for i in range(20) if int(m1[i]) > 0}
            assert all(int(m1[i]) in (0, int(m0[i])) for i in range(20))
            assert z1 == sum(int(m0[i]) for i in kept)
            pth = Fraction(round(p * 2**32), 2**32) * Z            # Theta's real value
            # brute force: try the levels t from the top; the answer is {mass >= t}
            # for the first level whose set reaches top_p.
            for t in sorted({int(x) for x in m0 if x > 0}, reverse=True):
                cand = {i for i in range(20) if int(m0[i]) >= t}
                if sum(int(m0[i]) for i in cand) >= pth:
                    break
            assert kept == cand
            assert prev_kept <= kept                       # monotone in top_p
            prev_kept = kept


# ------------------------------------------------------------------ sampling (R8), Eq. 3
def test_top_k_hand_examples(orc):
    """Reading R5k (P:202 'any top-p/top-k filtering'): keep the top_k heaviest masses,
    tie-closed.  (5,3,2), top_k 2 -> (0.625, 0.375, 0) after renormalisation; ties (4,4,4,1):
    top_k 1 or 2 keeps the whole tie group; top_k 0 or >= V is the identity."""
    for scale in (1, 1 << 20, 1 << 40):
        m, z = orc.top_k_filter(np.array([5, 3, 2], dtype=np.uint64) * np.uint64(scale), 2)
        assert [Fraction(int(x), z) for x in m] == [Fraction(5, 8), Fraction(3, 8), 0]
    for kk in (1, 2, 3):
        m, z = orc.top_k_filter(np.array([4, 4, 1, 4], dtype=np.uint64), kk)
        assert list(m) == [4, 4, 0, 4] and z == 12
    m, z = orc.top_k_filter(np.array([4, 4, 1, 4], dtype=np.uint64), 4)
    assert list(m) == [4, 4, 1, 4] and z == 13
    m, z = orc.top_k_filter(np.array([7, 0, 2], dtype=np.uint64), 0)
    assert list(m) == [7, 0, 2] and z == 9


def test_top_k_properties_random(orc):
    """Tie-closed top-k on random masses (many ties): every mass is kept or zeroed; the kept
    set is a top set of the mass order (each kept mass > each dropped one); if anything was
    dropped it has >= top_k members and is minimal (fewer than top_k masses exceed its
    lightest level); filtering twice changes nothing (SPEC S:96's idempotence holds for
    top-k)."""
    rng = np.random.default_rng(5)
    for _ in range(300):
        V = int(rng.integers(1, 40))
        mass = rng.integers(0, 6, V).astype(np.uint64) * np.uint64(1 << int(rng.integers(0, 40)))
        kk = int(rng.integers(0, V + 3))
        m, z = orc.top_k_filter(mass, kk)
        assert ((m == mass) | (m == 0)).all() and z == int(m.sum())
        kept, dropped = mass[m > 0], mass[(m == 0) & (mass > 0)]
        if kk <= 0 or kk >= V:
            assert len(dropped) == 0
        if len(dropped):
            assert len(kept) >= kk and dropped.max() < kept.min()
            assert int((mass > kept.min()).sum()) < kk
        m2, z2 = orc.top_k_filter(m, kk)
        assert (m2 == m).all() and z2 == z


def test_top_k_then_top_p_order(orc):
    """SPEC S:74 / S:99 filter order, top-k THEN top-p, on a row whose masses are ~(4,3,2,1)
    (logits ln 4, ln 3, ln 2, 0): top_k 2 renormalises to ~(4/7, 3/7) and top_p 0.5 then keeps
    only token 0 (4/7 >= 0.5); the opposite order would keep {0, 1} (0.4 < 0.5).  top_k 1
    equals greedy's support (argmax), top_k = V equals no filter."""
    row = bf16_row([math.log(4), math.log(3), math.log(2), 0.0])
    d = orc.row_dist(row, 1.0, 0.5, 2)
    assert [int(x) > 0 for x in d.mass] == [True, False, False, False] and d.z == int(d.mass[0])
    d = orc.row_dist(row, 1.0, 1.0, 2)
    assert [int(x) > 0 for x in d.mass] == [True, True, False, False]
    d = orc.row_dist(row, 1.0, 0.5, 0)
    assert [int(x) > 0 for x in d.mass] == [True, True, False, False]
    full = orc.row_dist(row, 1.0)
    assert (orc.row_dist(row, 1.0, 1.0, 4).mass == full.mass).all()
    assert int(np.argmax(orc.row_dist(row, 1.0, 1.0, 1).mass)) == orc.row_dist(row, 0.0).greedy


def test_inverse_cdf_spec_example(orc):
    """(0.5,0.5): u = 0.25 -> 0, u = 0.75 -> 1; S:85 degenerate (0,1,0) -> 1."""
    mass = [1, 1]
    assert orc.sample_index(mass, -1, orc.uniform_floor([0x40000000, 0, 0, 0], 2)) == 0
    assert orc.sample_index(mass, -1, orc.uniform_floor([0xC0000000, 0, 0, 0], 2)) == 1
    for U in range(1):
        assert orc.sample_index([0, 1, 0], -1, U) == 1


def test_residual_spec_example_exhaustive(orc):
    """S:232-233 (Eq. 3): (0.5,0.3,0.2) reject 0 -> (0, 0.6, 0.4); (0.5,0.5) reject 1 -> (1,0).
    Exact: enumerate every U in [0, Z - mass(excl))."""
    def dist(mass, excl):
        zx = sum(mass) - mass[excl]
        cnt = [0] * len(mass)
        for U in range(zx):
            cnt[orc.sample_index(mass, excl, U)] += 1
        return [Fraction(c, zx) for c in cnt]

    assert dist([5, 3, 2], 0) == [0, Fraction(3, 5), Fraction(2, 5)]
    assert dist([1, 1], 1) == [1, 0]


def test_per_token_marginal_identity(orc):
    """S:267 / P:211: p(d) 1[x=d] + (1 - p(d)) r(x) = p(x), exactly, by enumerating the
    accept draw and the residual draw on random small integer masses."""
    rng = np.random.default_rng(6)
    for _ in range(60):
        V = int(rng.integers(2, 6))
        mass = [int(x) for x in rng.integers(0, 7, V)]
        if sum(mass) == 0:
            mass[0] = 1
        Z = sum(mass)
        for d in range(V):
            P = [Fraction(0)] * V
            P[d] += Fraction(mass[d], Z)            # accept region U < mass(d)
            zx = Z - mass[d]
            if zx:
                for U in range(zx):                 # residual draw
                    P[orc.sample_index(mass, d, U)] += Fraction(Z - mass[d], Z) / zx
            assert P == [Fraction(m, Z) for m in mass]


# ------------------------------------------------------------------ Alg. 1 step
def onehot_row(V, tok):
    v = np.full(V, -np.inf, dtype=np.float32)
    v[tok] = 0.0
    return bf16_row(v)


def test_degenerate_rows_all_accepted(orc):
    """p_t(d_t) = 1 on every row -> all accepted, q + 1 emitted (bonus)."""
    V, k = 16, 4
    draft = [3, 5, 7, 9]
    rows = [onehot_row(V, t) for t in draft] + [onehot_row(V, 11)]
    for uid in range(20):
        out = orc.verify_one(rows, 1.0, 1.0, 9, uid, 0, 100, -1, False, draft, k)
        assert out.tokens == draft + [11] and out.accepted == 4 and out.rows_used == 5


def test_zero_mass_draft_rejected_first(orc):
    """p(d_1) = 0 -> rejected at 1, emitted token drawn from p_1 itself."""
    V = 8
    rng = np.random.default_rng(7)
    base = rng.normal(0, 1, V).astype(np.float32)
    base[2] = -np.inf
    row0 = bf16_row(base)
    rows = [row0] + [bf16_row(rng.normal(0, 1, V)) for _ in range(3)]
    for uid in range(50):
        out = orc.verify_one(rows, 1.0, 1.0, 1, uid, 5, 100, -1, False, [2, 1, 1], 3)
        assert out.accepted == 0 and len(out.tokens) == 1 and out.tokens[0] != 2
        assert out.rows_used == 1  # lazy: rows after the first rejection untouched


def test_step_token_distribution_chi_square(orc):
    """First emitted token of a step is distributed as p_0 (P:211 losslessness):
    chi-square over 20000 uids with a draft token of moderate probability."""
    from scipy.stats import chisquare

    V = 6
    rng = np.random.default_rng(8)
    rows = [bf16_row(rng.normal(0, 1, V)) for _ in range(3)]
    d0 = orc.row_dist(rows[0], 1.0)
    p = d0.mass.astype(np.float64) / d0.z
    n = 20000
    cnt = np.zeros(V)
    for uid in range(n):
        out = orc.verify_one(rows, 1.0, 1.0, 123, uid, 0, 100, -1, False, [1, 2], 2)
        cnt[out.tokens[0]] += 1
    assert chisquare(cnt, p * n).pvalue > 1e-3


def test_closed_form_acceptance_length(orc):
    """S:244 / S:594: i.i.d. per-row acceptance probability rho -> E[emitted] =
    sum_{i=0}^{q} rho^i (geometric truncation), and the accepted-count histogram matches."""
    V, q = 32, 4
    vals = np.zeros(V, dtype=np.float32)
    vals[0] = 2.0
    row = bf16_row(vals)
    d = orc.row_dist(row, 1.0)
    rho = int(d.mass[0]) / d.z
    rows = [row] * (q + 1)
    n = 20000
    emitted = np.zeros(n)
    acc_hist = np.zeros(q + 1)
    for uid in range(n):
        out = orc.verify_one(rows, 1.0, 1.0, 77, uid, 0, 1000, -1, False, [0] * q, q)
        emitted[uid] = len(out.tokens)
        acc_hist[out.accepted] += 1
    expect = sum(rho**i for i in range(q + 1))
    assert abs(emitted.mean() - expect) / expect < 0.01
    probs = np.array([rho**a * (1 - rho) for a in range(q)] + [rho**q])
    sd = np.sqrt(n * probs * (1 - probs))
    assert np.all(np.abs(acc_hist - n * probs) < 4 * sd + 1)


def test_accepted_eos_stops_block(orc):
    """an accepted EOS ends the block; no bonus token."""
    V, eos = 8, 7
    rows = [onehot_row(V, 1), onehot_row(V, eos), onehot_row(V, 2), onehot_row(V, 3)]
    out = orc.verify_one(rows, 1.0, 1.0, 1, 0, 0, 100, eos, False, [1, eos, 2], 3)
    assert out.tokens == [1, eos] and out.accepted == 2 and out.rows_used == 2


def test_max_len_clamp_and_finished(orc):
    """Reading L6: q <= max_len - pos - 1; finished or pos >= max_len emits nothing."""
    V = 8
    rows = [onehot_row(V, t) for t in [1, 2, 3, 4, 5]]
    out = orc.verify_one(rows, 1.0, 1.0, 1, 0, 8, 10, -1, False, [1, 2, 3, 4], 4)
    assert out.tokens == [1, 2] and out.accepted == 1   # q clamped to 1, bonus from row 1
    out = orc.verify_one(rows, 1.0, 1.0, 1, 0, 10, 10, -1, False, [1, 2], 4)
    assert out.tokens == []
    out = orc.verify_one(rows, 1.0, 1.0, 1, 0, 0, 10, -1, True, [1, 2], 4)
    assert out.tokens == []


def test_greedy_accepted_length_is_lcp(orc):
    """north_star (2): under greedy decoding the accepted length equals the brute-force
    longest common prefix of the draft and the greedy (argmax) continuation."""
    rng = np.random.default_rng(9)
    V, k = 12, 6
    for trial in range(200):
        rows = [bf16_row(rng.normal(0, 2, V)) for _ in range(k + 1)]
        greedy = [int(np.argmax(bf16_bits_to_f32(r))) for r in rows]
        draft = [g if rng.random() < 0.7 else int(rng.integers(0, V)) for g in greedy[:k]]
        lcp = 0
        while lcp < k and draft[lcp] == greedy[lcp]:
            lcp += 1
        out = orc.verify_one(rows, 0.0, 1.0, 5, trial, 0, 1000, -1, False, draft, k)
        assert out.accepted == lcp
        assert out.tokens == greedy[: lcp + 1]


# ------------------------------------------------------------------ full rollouts
def _markov_setup(V, seed):
    """Order-1 Markov target over V tokens: row for prev token x is rows[x]."""
    rng = np.random.default_rng(seed)
    return [bf16_row(rng.normal(0, 1.0, V)) for _ in range(V)]


def _run_spec_rollouts(orc, rows_by_prev, pools, n, L, k, T, eos, prompt_last=0, seed=11):
    from oracle.rollout import OracleRollout, run_rollouts

    def row_fn(P, positions, prevs, uid=0):
        return [rows_by_prev[p] for p in prevs]

    ros = [OracleRollout(prompt=0, uid=u, context=[prompt_last], max_len=L) for u in range(n)]
    run_rollouts(ros, pools, row_fn, k=k, M=8, Lmin=1, T=T, top_p=1.0, seed=seed, eos=eos)
    return ros


def test_lossless_sequence_distribution_chi_square(orc):
    """S:591-592 / P:211 'exactly preserves the target rollout distribution': V=4 order-1
    Markov target, L=5, K=2, a 6-sequence pool.  The empirical distribution of whole
    speculative rollouts matches the autoregressive product distribution (exact masses)."""
    from scipy.stats import chisquare

    V, L, k, eos = 4, 5, 2, 3
    rows = _markov_setup(V, 12)
    pools = {0: [[0, 1, 2, 1, 0], [1, 2, 1, 2], [2, 2, 0, 1], [0, 0, 1, 2, 3], [1, 1, 1], [2, 0]]}
    n = 30000
    ros = _run_spec_rollouts(orc, rows, pools, n, L, k, 1.0, eos)
    assert sum(len(s[2]) > 0 for r in ros for s in r.steps) > n  # drafts were used
    probs = {}
    dists = [orc.row_dist(r, 1.0) for r in rows]

    def expand(prefix, prev, pr):
        if len(prefix) == L or (prefix and prefix[-1] == eos):
            probs[tuple(prefix)] = pr
            return
        d = dists[prev]
        for x in range(V):
            if int(d.mass[x]):
                expand(prefix + [x], x, pr * Fraction(int(d.mass[x]), d.z))

    expand([], 0, Fraction(1))
    keys = sorted(probs)
    idx = {kk: i for i, kk in enumerate(keys)}
    cnt = np.zeros(len(keys))
    for r in ros:
        cnt[idx[tuple(r.generated)]] += 1
    exp = np.array([float(probs[kk]) for kk in keys]) * n
    big = exp >= 5
    obs = np.append(cnt[big], cnt[~big].sum())
    ex = np.append(exp[big], exp[~big].sum())
    assert chisquare(obs, ex).pvalue > 1e-3


@pytest.mark.parametrize("T,top_p", [(1.0, 1.0), (0.7, 1.0), (1.0, 0.8), (0.0, 1.0)])
def test_lossless_exact_enumeration(orc, T, top_p):
    """S:591 / SURVEY c.6 'losslessness, exact' (P:211 'exactly preserves the target rollout
    distribution'): V=4 order-1 Markov target, L=5, K=2, EOS=3, a 6-sequence pool.  Every
    branch of every speculative step is enumerated with the ideal uniform (accept d with
    mass'(d)/Z', residual x with mass'_x/(Z'-mass'(d)), bonus x with mass'_x/Z'), and each branch
    is confirmed by driving the oracle's step (orc_verify_one_r) with a uniform inside that
    branch's interval.  The distribution over whole rollouts EQUALS the autoregressive product
    of the same rows (Fractions: TV = 0), so a dropped, misplaced or mis-indexed term anywhere in
    the step (row j vs j-1, the excluded token, the bonus row, the EOS stop, the length clamp)
    fails it."""
    TWO128 = 1 << 128
    V, L, k, eos, M = 4, 5, 2, 3, 8
    rows = _markov_setup(V, 12)
    pool = [[0, 1, 2, 1, 0], [1, 2, 1, 2], [2, 2, 0, 1], [0, 0, 1, 2, 3], [1, 1, 1], [2, 0]]
    dists = [orc.row_dist(r, T, top_p) for r in rows]
    mass_of = [[int(x) for x in d.mass] for d in dists]

    def r_inside(C, Z):  # the smallest r128 with floor(r * Z / 2^128) == C (C < Z)
        return -(-C * TWO128 // Z)

    def branches(draft, prevs):
        pr = Fraction(1)
        acc_r, smp_r = [0] * (k + 1), [0] * (k + 1)
        q = len(draft)
        for j in range(q + 1):
            mass, Z = mass_of[prevs[j]], dists[prevs[j]].z
            if j < q:
                d = draft[j]
                if mass[d] < Z:  # rejection at row j, then the residual sample (Eq. 3)
                    Zx, C = Z - mass[d], 0
                    for x in range(V):
                        if x != d and mass[x]:
                            ra, rs = list(acc_r), list(smp_r)
                            ra[j], rs[j] = TWO128 - 1, r_inside(C, Zx)
                            yield draft[:j] + [x], pr * Fraction(Z - mass[d], Z) * Fraction(mass[x], Zx), ra, rs
                            C += mass[x]
                if mass[d] == 0:
                    return
                pr *= Fraction(mass[d], Z)  # accepted (Eq. 2): U = 0 < mass(d)
                if d == eos:
                    yield draft[:j + 1], pr, list(acc_r), list(smp_r)
                    return
            else:  # bonus (or the plain sample when q = 0)
                C = 0
                for x in range(V):
                    if mass[x]:
                        rs = list(smp_r)
                        rs[q] = r_inside(C, Z)
                        yield draft + [x], pr * Fraction(mass[x], Z), list(acc_r), rs
                        C += mass[x]

    spec, steps_with_drafts = {}, [0]

    def run(gen, pr):
        if len(gen) == L or (gen and gen[-1] == eos):
            spec[tuple(gen)] = spec.get(tuple(gen), Fraction(0)) + pr
            return
        ctx = [0] + gen
        draft, _ = orc.lookup(pool, ctx, M, 1, k)
        draft = draft[:max(0, min(len(draft), L - len(gen) - 1))]
        steps_with_drafts[0] += bool(draft)
        prevs = [ctx[-1]] + draft
        for toks, p, ra, rs in branches(draft, prevs):
            out = orc.verify_one_r([rows[x] for x in prevs], T, top_p, len(gen), L, eos, draft, k, ra, rs)
            assert out.tokens == toks, (gen, draft, toks, out.tokens)
            run(gen + toks, pr * p)

    run([], Fraction(1))
    ar = {}

    def expand(prefix, prev, p):
        if len(prefix) == L or (prefix and prefix[-1] == eos):
            ar[tuple(prefix)] = p
            return
        for x in range(V):
            if mass_of[prev][x]:
                expand(prefix + [x], x, p * Fraction(mass_of[prev][x], dists[prev].z))

    expand([], 0, Fraction(1))
    assert steps_with_drafts[0] >= 2  # the pool drafted (on many branches at T > 0, top_p = 1)
    assert sum(spec.values()) == 1
    assert spec == ar  # total variation 0


def test_empty_pool_is_plain_decoding(orc):
    """north_star (3) / S:252: with an empty pool every step is one plain sample drawn
    with counter (t, SAMPLE); under T = 0 this is the argmax chain (numpy argmax)."""
    V, L = 6, 12
    rows = _markov_setup(V, 13)
    ros = _run_spec_rollouts(orc, rows, {}, 5, L, 3, 0.0, -1)
    for r in ros:
        chain, prev = [], 0
        for _ in range(L):
            prev = int(np.argmax(bf16_bits_to_f32(rows[prev])))
            chain.append(prev)
        assert r.generated == chain and len(r.steps) == L
    ros = _run_spec_rollouts(orc, rows, {}, 3, L, 3, 1.0, -1, seed=99)
    for r in ros:
        prev = 0
        for t, x in enumerate(r.generated):
            d = orc.row_dist(rows[prev], 1.0)
            U = orc.uniform_floor(orc.draw_r128(99, r.uid, t, 1), d.z)
            c = np.cumsum(d.mass.astype(object))
            assert x == int(np.argmax(c > U))
            prev = x


# ------------------------------------------------------------------ lookup
def _trie_lookup(pool, ctx, M, Lmin, K, tau_q=0):
    """Independent route to the lookup definition: count every window of the pool with
    a Python Counter (a depth-bounded suffix trie), then anchor + greedy descent; tau_q > 0:
    stop before a child whose count is below tau_q / 2^32 of its node's count (reading C1)."""
    from collections import Counter

    D = M + K + 1
    cnt, cont = Counter(), Counter()
    for s in pool:
        for i in range(len(s)):
            for l in range(1, min(D, len(s) - i) + 1):
                w = tuple(s[i:i + l])
                cnt[w] += 1
                if i + l < len(s):
                    cont[w] += 1
    mstar = 0
    for m in range(min(M, len(ctx)), Lmin - 1, -1):
        if cont[tuple(ctx[len(ctx) - m:])] >= 1:
            mstar = m
            break
    if mstar == 0:
        return [], 0
    w = list(ctx[len(ctx) - mstar:])
    out = []
    for _ in range(K):
        kids = {w2[-1]: c for w2, c in cnt.items() if len(w2) == len(w) + 1 and list(w2[:-1]) == w}
        if not kids:
            break
        best = min(kids, key=lambda t: (-kids[t], t))
        if kids[best] * (1 << 32) < tau_q * cnt[tuple(w)]:
            break
        out.append(best)
        w.append(best)
    return out, mstar


def test_lookup_spec_examples(orc):
    """S:154."""
    pool = [[1, 2, 3], [1, 2, 3], [1, 2, 5]]
    d, m = orc.lookup(pool, [9, 1, 2], 8, 1, 4)
    assert d[0] == 3 and m == 2 and d == [3]
    d, m = orc.lookup([[7, 8]], [4, 4, 7], 8, 1, 4)
    assert d == [8] and m == 1
    d, m = orc.lookup(pool, [9, 9, 9], 8, 1, 4)
    assert d == [] and m == 0
    d, m = orc.lookup([], [1, 2], 8, 1, 4)
    assert d == [] and m == 0


def test_lookup_anchor_needs_continuation(orc):
    """Reading L2: a suffix that occurs only at sequence ends does not anchor; the
    longest suffix WITH a continuation does."""
    pool = [[5, 6, 7], [6, 1]]
    d, m = orc.lookup(pool, [5, 6], 8, 1, 3)
    assert m == 2 and d == [7]
    d, m = orc.lookup(pool, [9, 6, 7], 8, 1, 3)   # "6 7" and "7" only at ends
    assert m == 0 and d == []
    d, m = orc.lookup([[1, 2], [3, 1, 4]], [3, 9, 3, 1], 8, 1, 3)  # "3 1" has cont via seq 2
    assert m == 2 and d == [4]


def test_lookup_vs_trie_random(orc):
    """200 random pools x several prefixes, oracle == independent trie lookup."""
    rng = np.random.default_rng(10)
    for t in range(200):
        V = int(rng.integers(2, 6))
        pool = [list(rng.integers(0, V, int(rng.integers(0, 12)))) for _ in range(int(rng.integers(0, 5)))]
        pool = [[int(x) for x in s] for s in pool]
        for _ in range(5):
            ctx = [int(x) for x in rng.integers(0, V, int(rng.integers(1, 10)))]
            M = int(rng.integers(1, 6))
            Lmin = int(rng.integers(1, 3))
            K = int(rng.integers(0, 5))
            assert orc.lookup(pool, ctx, M, Lmin, K) == _trie_lookup(pool, ctx, M, Lmin, K)


def test_lookup_invariants(orc):
    """The draft is the continuation of some occurrence of anchor+draft in one sequence;
    the anchor is maximal (m*+1 has no continuation)."""
    rng = np.random.default_rng(11)
    for _ in range(200):
        pool = [[int(x) for x in rng.integers(0, 4, 15)] for _ in range(4)]
        ctx = [int(x) for x in rng.integers(0, 4, 10)]
        d, m = orc.lookup(pool, ctx, 6, 1, 5)
        if m == 0:
            continue
        s = ctx[-m:] + d
        assert any(seq[i:i + len(s)] == s for seq in pool for i in range(len(seq)))
        if m < 6:
            w = ctx[-(m + 1):]
            assert not any(seq[i:i + len(w)] == w and i + len(w) < len(seq)
                           for seq in pool for i in range(len(seq)))


# ------------------------------------------------------------------ n-gram drafter (f4)
def test_ngram_hand_examples(orc):
    """Reading N1 ('a linear match of repeated token sequences ... the candidate with
    the longest common prefix'): the longest suffix wins; among its occurrences the first in
    pool order; the draft is cut at its sequence's end; a terminal-only match does not anchor;
    n is bounded by n_max and n_min."""
    pool = [[1, 2, 3, 4], [9, 1, 2, 5], [7, 7, 1, 2]]
    assert orc.lookup_ngram(pool, [8, 1, 2], 1, 4, 3) == ([3, 4], 2)      # first occurrence
    assert orc.lookup_ngram(pool, [9, 1, 2], 1, 4, 3) == ([5], 3)         # longest wins
    assert orc.lookup_ngram(pool, [9, 1, 2], 1, 2, 3) == ([3, 4], 2)      # n_max caps n
    assert orc.lookup_ngram(pool, [6, 4], 1, 4, 3) == ([], 0)             # 4 only ends a sequence
    assert orc.lookup_ngram(pool, [7, 7], 1, 4, 5) == ([1, 2], 2)
    assert orc.lookup_ngram(pool, [5, 7], 2, 4, 3) == ([], 0)             # n_min 2: no match
    assert orc.lookup_ngram(pool, [5, 7], 1, 4, 3) == ([7, 1, 2], 1)      # K = 3 tokens
    assert orc.lookup_ngram([], [1], 1, 4, 3) == ([], 0)


def test_ngram_vs_backward_match_scan(orc):
    """Independent route: for every pool position e (followed by a token) the backward match
    length against the context, then the best (length desc, position asc); 300 random pools."""
    rng = np.random.default_rng(17)
    for _ in range(300):
        vocab = int(rng.integers(2, 6))
        pool = [list(rng.integers(0, vocab, int(rng.integers(0, 12)))) for _ in range(int(rng.integers(0, 5)))]
        ctx = list(rng.integers(0, vocab, int(rng.integers(1, 10))))
        n_min, n_max, K = int(rng.integers(1, 3)), int(rng.integers(3, 8)), int(rng.integers(1, 6))
        best = (0, 0, None)
        flat = [(s, i) for s, seq in enumerate(pool) for i in range(len(seq))]
        for pos, (s, e) in enumerate(flat):
            seq = pool[s]
            if e + 1 >= len(seq):
                continue
            n = 0
            while n < min(n_max, len(ctx)) and e - n >= 0 and seq[e - n] == ctx[-1 - n]:
                n += 1
            if n >= n_min and n > best[0]:
                best = (n, pos, seq[e + 1:e + 1 + K])
        want = (best[2], best[0]) if best[2] is not None else ([], 0)
        assert orc.lookup_ngram(pool, ctx, n_min, n_max, K) == ([int(x) for x in want[0]], want[1])


# ------------------------------------------------------------------ confidence-scored drafts (C1)
def test_lookup_conf_hand_example(orc):
    """Reading C1 on the S:154 pool: after the anchor "1 2" (3 occurrences) the greedy child 3
    has probability 2/3, so it is drafted for tau <= 2/3 and not above; tau = 0 is the plain
    lookup; a unique continuation (probability 1) survives tau = 1."""
    pool = [[1, 2, 3], [1, 2, 3], [1, 2, 5]]
    assert orc.lookup(pool, [9, 1, 2], 8, 1, 4, 0.0) == orc.lookup(pool, [9, 1, 2], 8, 1, 4)
    assert orc.lookup(pool, [9, 1, 2], 8, 1, 4, 0.5) == ([3], 2)
    assert orc.lookup(pool, [9, 1, 2], 8, 1, 4, 2.0 / 3.0 - 1e-9) == ([3], 2)
    assert orc.lookup(pool, [9, 1, 2], 8, 1, 4, 0.7) == ([], 2)
    # "7 8" occurs once and continues: every step has probability 1
    assert orc.lookup([[7, 8, 9, 10, 11]], [7, 8], 8, 1, 3, 1.0) == ([9, 10, 11], 2)
    # a window that also ends a sequence: cnt(w) counts that occurrence (2 of 3 continue with 4)
    assert orc.lookup([[3, 4], [3, 4], [3]], [3], 8, 1, 2, 0.6) == ([4], 1)
    assert orc.lookup([[3, 4], [3, 4], [3]], [3], 8, 1, 2, 0.7) == ([], 1)


def test_lookup_conf_vs_trie_random(orc):
    """Random pools: the thresholded oracle == the independent trie with the same rule, the
    drafts are prefixes of the plain drafts and shrink as tau grows, and at tau = 1 every
    drafted token is the continuation of ALL occurrences of its window."""
    rng = np.random.default_rng(11)
    for t in range(150):
        V = int(rng.integers(2, 5))
        pool = [[int(x) for x in rng.integers(0, V, int(rng.integers(0, 14)))] for _ in range(int(rng.integers(0, 6)))]
        for _ in range(4):
            ctx = [int(x) for x in rng.integers(0, V, int(rng.integers(1, 9)))]
            M, Lmin, K = int(rng.integers(1, 6)), int(rng.integers(1, 3)), int(rng.integers(1, 6))
            plain = orc.lookup(pool, ctx, M, Lmin, K)
            prev = plain[0]
            for tau in (0.25, 0.5, 0.75, 1.0):
                got = orc.lookup(pool, ctx, M, Lmin, K, tau)
                assert got == _trie_lookup(pool, ctx, M, Lmin, K, orc.tau_fixed(tau))
                assert got[1] == plain[1] and got[0] == prev[:len(got[0])]
                prev = got[0]
            w = ctx[len(ctx) - plain[1]:] if plain[1] else []
            for tok in prev:  # tau = 1: deterministic continuations only
                occ = [(s, i) for s in pool for i in range(len(s) - len(w) + 1) if s[i:i + len(w)] == w]
                assert occ and all(i + len(w) < len(s) and s[i + len(w)] == tok for s, i in occ)
                w = w + [tok]
