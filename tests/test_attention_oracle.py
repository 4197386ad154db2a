"""Pins of the attention oracle (oracle/attention.py): each check compares it
with something the mathematics fixes, never with the CUDA path.  CPU only."""
import numpy as np
import pytest

from oracle.attention import attention_batch, attention_request
from workloads import bf16_bits_to_f32, f32_to_bf16_bits
from workloads.attn import PAGE, logical_kv, make_attn_batch


def _bits(x):
    return f32_to_bf16_bits(np.asarray(x, dtype=np.float32))


def test_equal_keys_give_the_mean_of_values():
    """All keys equal -> uniform weights over the causal window -> mean of those values."""
    rng = np.random.default_rng(1)
    L, q_len, H_q, H_kv, d = 37, 4, 6, 2, 8
    k = np.broadcast_to(rng.normal(size=(1, H_kv, d)), (L, H_kv, d))
    v = rng.normal(size=(L, H_kv, d))
    q = rng.normal(size=(q_len, H_q, d))
    vb = bf16_bits_to_f32(_bits(v)).astype(np.float64)
    o = attention_request(_bits(q), _bits(k), _bits(v), H_kv)
    for i in range(q_len):
        p = L - q_len + i
        for h in range(H_q):
            np.testing.assert_allclose(o[i, h], vb[: p + 1, h // (H_q // H_kv)].mean(axis=0), rtol=1e-12, atol=1e-12)


def test_dominant_key_selects_its_value():
    """One key aligned with the query and a large scale: the softmax is one-hot on it."""
    d = 16
    q = np.zeros((1, 1, d)); q[0, 0, 3] = 1.0
    k = np.zeros((20, 1, d)); k[7, 0, 3] = 1.0
    v = np.arange(20 * d, dtype=np.float64).reshape(20, 1, d) / 64.0
    o = attention_request(_bits(q), _bits(k), _bits(v), 1, scale=200.0)
    np.testing.assert_allclose(o[0, 0], bf16_bits_to_f32(_bits(v))[7, 0], rtol=0, atol=1e-70)


def test_single_query_equals_torch_sdpa_and_gqa_mapping():
    """q_len = 1 (a plain decode token sees the whole context): torch's scaled-dot-product
    attention in fp64 on CPU (a library routine) with K/V heads repeated G times."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(2)
    L, H_q, H_kv, d = 50, 8, 2, 16
    q, k, v = rng.normal(size=(1, H_q, d)), rng.normal(size=(L, H_kv, d)), rng.normal(size=(L, H_kv, d))
    o = attention_request(_bits(q), _bits(k), _bits(v), H_kv)
    f = lambda x: torch.from_numpy(bf16_bits_to_f32(_bits(x)).astype(np.float64))  # noqa: E731
    qt = f(q).permute(1, 0, 2)[None]                                    # [1, H_q, 1, d]
    kt = f(k).permute(1, 0, 2).repeat_interleave(H_q // H_kv, 0)[None]  # [1, H_q, L, d]
    vt = f(v).permute(1, 0, 2).repeat_interleave(H_q // H_kv, 0)[None]
    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt)[0].permute(1, 0, 2).numpy()
    np.testing.assert_allclose(o, ref, rtol=1e-12, atol=1e-12)


def test_causal_window_of_the_query_block():
    """Query token i of a q_len block sees keys 0 .. L - q_len + i: changing later keys / values
    leaves it unchanged, changing an earlier one changes it (P:236-241 speculative queries are
    causal prefill-like rows)."""
    rng = np.random.default_rng(3)
    L, q_len, H_q, H_kv, d = 30, 5, 4, 1, 8
    q, k, v = rng.normal(size=(q_len, H_q, d)), rng.normal(size=(L, H_kv, d)), rng.normal(size=(L, H_kv, d))
    o = attention_request(_bits(q), _bits(k), _bits(v), H_kv)
    for i in range(q_len):
        p = L - q_len + i
        k2, v2 = k.copy(), v.copy()
        k2[p + 1:] += 3.0
        v2[p + 1:] -= 2.0
        o2 = attention_request(_bits(q), _bits(k2), _bits(v2), H_kv)
        np.testing.assert_array_equal(o2[i], o[i])
        if p + 1 < L:
            assert not np.array_equal(o2[q_len - 1], o[q_len - 1])


def test_paged_batch_gathers_each_requests_pages():
    """The batch oracle on a paged cache (shuffled pages, ragged lengths) equals the per-request
    oracle on contiguous K/V rebuilt independently from the page table."""
    b = make_attn_batch(4, [1, 5, 2], [PAGE + 3, 2 * PAGE, 7], H_q=4, H_kv=2, d=8)
    o = attention_batch(b)
    for r in range(3):
        L = int(b.ctx_len[r])
        k = np.concatenate([b.k_cache[b.page_table[r, i]].transpose(1, 0, 2) for i in range((L + PAGE - 1) // PAGE)])[:L]
        v = np.concatenate([b.v_cache[b.page_table[r, i]].transpose(1, 0, 2) for i in range((L + PAGE - 1) // PAGE)])[:L]
        kk, vv = logical_kv(b, r)
        assert np.array_equal(k, kk) and np.array_equal(v, vv)
        r0, r1 = int(b.q_off[r]), int(b.q_off[r + 1])
        np.testing.assert_array_equal(o[r0:r1], attention_request(b.q[r0:r1], k, v, 2))


# ------------------------------------------------------------------ f3 LM-head logits oracle
def test_lm_head_one_hot_weights_copy_the_hidden_state():
    """W[v] = s_v * e_{v mod d}: logits[r, v] = bf16(s_v * h[r, v mod d]) exactly (one product,
    no sum), including the round-to-nearest-even of the product."""
    from oracle.lm_head import lm_head_logits

    rng = np.random.default_rng(7)
    rows, d, V = 5, 16, 48
    h = _bits(rng.normal(size=(rows, d)))
    scale = np.array([1.0, 3.0, -0.375, 2.0 ** -7] * (V // 4))
    w = np.zeros((V, d))
    w[np.arange(V), np.arange(V) % d] = scale
    out = lm_head_logits(h, _bits(w))
    want = f32_to_bf16_bits((bf16_bits_to_f32(h)[:, np.arange(V) % d].astype(np.float64) * scale).astype(np.float32))
    np.testing.assert_array_equal(out, want)


def test_lm_head_rne_tie_and_row_stats():
    """A dot product landing exactly half-way between two bf16 values rounds to the even one;
    row statistics: max, the lowest index attaining it, -inf is not an error, NaN / +inf are."""
    from oracle.lm_head import lm_head_logits, row_stats

    # 1 + 2^-8 is half-way between 1 and 1 + 2^-7: ties to even (1.0); 1 + 3*2^-8 -> 1 + 2^-6
    h = _bits([[1.0, 2.0 ** -8]])
    w = _bits([[1.0, 1.0], [1.0, 3.0]])
    out = bf16_bits_to_f32(lm_head_logits(h, w))
    assert out[0, 0] == 1.0 and out[0, 1] == 1.0 + 2.0 ** -6
    m, am, bad = row_stats(_bits([[1.0, 5.0, 5.0, -np.inf], [-np.inf, -2.0, -np.inf, -3.0]]))
    assert list(m) == [5.0, -2.0] and list(am) == [1, 1] and not bad.any()
    nan_row = np.array([[0x3F80, 0x7FC0, 0x3F80]], dtype=np.uint16)
    inf_row = np.array([[0x3F80, 0x7F80, 0x3F80]], dtype=np.uint16)
    assert row_stats(nan_row)[2][0] and row_stats(inf_row)[2][0]
