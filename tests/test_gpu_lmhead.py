"""f3: the tcgen05 LM-head GEMM with the verify's first pass fused into its
epilogue, vs the oracle (oracle/lm_head.py) and vs the verify without the fused statistics.

Tolerance of the logits, from the arithmetic: products of bf16 values are exact in fp32 and the
d-term sums are accumulated in fp32 by the tensor cores in an order the oracle (fp64, one
rounding) does not reproduce.  The fp32 sum's absolute error is at most
gamma_d * sum_k |h_k||w_k| with gamma_d = d * 2^-24 (the standard recursive-summation bound), and
the final bf16 rounding adds at most one bf16 ulp of the result; so each GPU logit must be within
ulp(ref) + gamma_d * (|h| |W|^T) of the oracle's, and almost all must be equal.  The fused row statistics are checked
EXACTLY against the GPU's own logits (max, lowest argmax, NaN / +inf flag), and a verify given
them must emit exactly what it emits without them."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.lm_head import lm_head_logits, row_stats  # noqa: E402
from workloads import bf16_bits_to_f32, f32_to_bf16_bits  # noqa: E402
from workloads.attn import _vals  # noqa: E402

from tests.gpu_util import to_dev  # noqa: E402


def _inputs(rows, d, V, seed):
    h = f32_to_bf16_bits(_vals(seed, 21, rows * d, 1.0)).reshape(rows, d)
    w = f32_to_bf16_bits(_vals(seed, 22, V * d, 3.0 / np.sqrt(d))).reshape(V, d)
    return h, w


def _decode_key(k):
    k = np.asarray(k).astype(np.uint64)
    kb = (k >> np.uint64(32)).astype(np.uint32)
    bits = np.where(kb & 0x8000, kb & 0x7FFF, ~kb & 0xFFFF).astype(np.uint16)
    am = (np.uint64(0xFFFFFFFF) - (k & np.uint64(0xFFFFFFFF))).astype(np.int64)
    return bf16_bits_to_f32(bits), am


def _gpu(bs, h, w):
    lg, key, bad = bs.bs_lm_head_logits(to_dev(h.view(np.int16)), to_dev(w.view(np.int16)))
    torch.cuda.synchronize()
    return lg.cpu().numpy().view(np.uint16), key.cpu().numpy(), bad.cpu().numpy()


@pytest.mark.parametrize("rows,d,V", [(1, 64, 300), (37, 128, 4099), (200, 256, 1024), (130, 3584, 2500),
                                      (9, 3584, 151936)])
def test_lm_head_logits_and_fused_stats(bs, rows, d, V):
    h, w = _inputs(rows, d, V, rows + V)
    lg, key, bad = _gpu(bs, h, w)
    ref = lm_head_logits(h, w)
    g, r = bf16_bits_to_f32(lg).astype(np.float64), bf16_bits_to_f32(ref).astype(np.float64)
    hf, wf = np.abs(bf16_bits_to_f32(h).astype(np.float64)), np.abs(bf16_bits_to_f32(w).astype(np.float64))
    bound = np.abs(r) * 2.0 ** -7 + d * 2.0 ** -24 * (hf @ wf.T)
    assert (np.abs(g - r) <= bound).all(), float((np.abs(g - r) - bound).max())
    assert (lg == ref).mean() > 0.99
    # fused statistics: exactly the GPU logits' own (R1) and no NaN / +inf (R0)
    m, am = _decode_key(key)
    m_ref, am_ref, bad_ref = row_stats(lg)
    np.testing.assert_array_equal(m, m_ref)
    np.testing.assert_array_equal(am, am_ref)
    assert not bad.any() and not bad_ref.any()


def test_lm_head_stats_flag_nan_and_inf(bs):
    h, w = _inputs(5, 64, 700, 3)
    w[17] = 0x7FC0                   # NaN weights: column 17 is NaN in every row
    h[2, 0], w[400, 0] = 0x7F80, 0x3F80  # +inf in row 2 (h = +inf, w = 1 at column 400; others mixed)
    lg, key, bad = _gpu(bs, h, w)
    m_ref, am_ref, bad_ref = row_stats(lg)
    assert bad.all() and bad_ref.all()
    m, am = _decode_key(key)
    ok = np.isfinite(m_ref)
    np.testing.assert_array_equal(m[ok], m_ref[ok])


@pytest.mark.parametrize("T", [1.0, 0.0])
def test_verify_with_fused_stats_is_identical(bs, orc, T):
    """Logits from the LM head for n rollouts x (k+1) rows; the cluster verify with the fused row
    statistics (max pass skipped) == without them == the oracle on those logits."""
    n, k, d, V = 24, 4, 256, 4099
    h, w = _inputs(n * (k + 1), d, V, 11)
    # a few rows made peaked so drafts are accepted
    lg_d, key_d, bad_d = bs.bs_lm_head_logits(to_dev(h.view(np.int16)), to_dev(w.view(np.int16)))
    lg = lg_d.cpu().numpy().view(np.uint16).reshape(n, k + 1, V)
    argm = bf16_bits_to_f32(lg).argmax(axis=2)
    rng = np.random.default_rng(4)
    drafts = np.where(rng.random((n, k)) < 0.8, argm[:, :k], rng.integers(0, V, (n, k))).astype(np.int32)
    dlen = rng.integers(0, k + 1, n).astype(np.int32)
    res = []
    for use in (False, True):
        ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=8, max_rollouts=n, pool_capacity_tokens=16,
                         pool_capacity_seqs=4, seed=77)
        ctx.bsx_set_verify_kernel("cluster")
        if use:
            ctx.bsx_set_row_stats(key_d, bad_d)
        slots = to_dev(np.arange(n, dtype=np.int32))
        tail = np.full((n, 8), -1, np.int32)
        tail[:, -1] = 0
        uids = np.arange(n, dtype=np.int64) * 3 + 1
        ctx.bs_rollout_begin(slots, to_dev(uids), to_dev(np.zeros(n, np.int32)), to_dev(tail),
                             to_dev(np.full(n, 1000, np.int32)))
        ot = torch.zeros((n, k + 1), dtype=torch.int32, device="cuda")
        ol = torch.zeros(n, dtype=torch.int32, device="cuda")
        oa = torch.zeros(n, dtype=torch.int32, device="cuda")
        oz = torch.zeros((n, k + 1), dtype=torch.int64, device="cuda")
        ctx.bs_verify_step(slots, lg_d.view(-1), None, V, to_dev(drafts), to_dev(dlen), k, T, 1.0, ot, ol, oa,
                           None, oz)
        torch.cuda.synchronize()
        assert ctx.bs_sync_status() == 0
        res.append((ot.cpu().numpy(), ol.cpu().numpy(), oa.cpu().numpy(), oz.cpu().numpy()))
    for x, y in zip(*res):
        np.testing.assert_array_equal(x, y)
    ot, ol, oa, oz = res[1]
    for b in range(n):
        q = int(dlen[b])
        o = orc.verify_one([lg[b, j] for j in range(k + 1)], T, 1.0, 77, int(uids[b]), 0, 1000, -1, False,
                           [int(x) for x in drafts[b, :q]], k)
        assert [int(x) for x in ot[b, :ol[b]]] == o.tokens, b


def test_lm_head_full_size_sampled_rows(bs):
    """At the size the bench times (Qwen2.5-7B head, d 3584, V 151936, 2304 rows = 256 rollouts x
    9): the fused statistics of EVERY row equal the GPU logits' own, and sampled rows' logits are
    within the fp32-summation bound of the fp64 oracle."""
    rows, d, V = 2304, 3584, 151936
    mult_w = float(np.float32(3.0 / np.sqrt(d) / 147.8))
    w = torch.empty((V, d), dtype=torch.int16, device="cuda")
    bs.bsx_synth_attn_values(w, 22, mult_w)
    h = torch.empty((rows, d), dtype=torch.int16, device="cuda")
    bs.bsx_synth_attn_values(h, 21, float(np.float32(1.0 / 147.8)))
    lg, key, bad = bs.bs_lm_head_logits(h, w)
    torch.cuda.synchronize()
    f = lg.view(torch.bfloat16).float()
    m_dev = f.max(dim=1).values
    am_dev = (f == m_dev[:, None]).int().argmax(dim=1)
    m, am = _decode_key(key.cpu().numpy())
    np.testing.assert_array_equal(m, m_dev.cpu().numpy())
    np.testing.assert_array_equal(am, am_dev.cpu().numpy())
    assert not bad.cpu().numpy().any()
    sample = [0, 1, 777, 1500, rows - 1]
    hs = h[sample].cpu().numpy().view(np.uint16)
    wn = w.cpu().numpy().view(np.uint16)
    ref = lm_head_logits(hs, wn)
    g = bf16_bits_to_f32(lg[sample].cpu().numpy().view(np.uint16)).astype(np.float64)
    r = bf16_bits_to_f32(ref).astype(np.float64)
    hf, wf = np.abs(bf16_bits_to_f32(hs).astype(np.float64)), np.abs(bf16_bits_to_f32(wn).astype(np.float64))
    bound = np.abs(r) * 2.0 ** -7 + d * 2.0 ** -24 * (hf @ wf.T)
    assert (np.abs(g - r) <= bound).all()
    assert (lg[sample].cpu().numpy().view(np.uint16) == ref).mean() > 0.99


@pytest.mark.parametrize("zero_max", [False, True])
def test_lm_head_stats_ties_and_zero_maxima(bs, zero_max):
    """R1's ties: logits = s_r * w[v, 0] exactly (h one-hot), w[:, 0] drawn from a few values so
    the row maximum repeats within and across 32-column chunks and tiles; with zero_max the
    maximum is +-0 (the epilogue's per-element path).  The fused statistics must equal the GPU
    logits' own (lowest column of the maximum, order-key ties as R1)."""
    rows, d, V = 6, 64, 1000  # V not a multiple of 32: the last chunk straddles V
    rng = np.random.default_rng(7 + zero_max)
    h = np.zeros((rows, d), np.uint16)
    h[:, 0] = np.where(np.arange(rows) % 2 == 0, 0x3F80, 0xBF80)  # +1 / -1
    vals = np.array([-2.0, -1.0, 0.0] if zero_max else [-2.0, -1.0, 0.0, 1.0, 2.0], np.float32)
    w = f32_to_bf16_bits(_vals(5, 22, V * d, 0.5)).reshape(V, d)
    w[:, 0] = f32_to_bf16_bits(rng.choice(vals, V).astype(np.float32))
    if zero_max:
        h[1::2, 0] = 0x3F80  # every row +1: maximum 0
    lg, key, bad = _gpu(bs, h, w)
    m_ref, am_ref, bad_ref = row_stats(lg)
    m, am = _decode_key(key)
    np.testing.assert_array_equal(m, m_ref)
    np.testing.assert_array_equal(am, am_ref)
    assert not bad.any() and not bad_ref.any()
