"""f2 parity: the tcgen05 unified attention kernel (through the C-ABI) vs the
fp64 oracle (oracle/attention.py) on the same seeded paged-KV batches.

Tolerance, from the arithmetic: Q.K^T is exact bf16 products accumulated in fp32 (relative error
~1e-6); the softmax weights P are rounded to bf16 before the P.V tensor-core product (relative
error <= 2^-9 each) and the row sum uses the same rounded P, so |O - O_ref| <= 2^-9 * max|v|;
the output is rounded to bf16 (2^-9 relative).  The test bound is
|O - O_ref| <= 2^-8 * max|v of the request| + 2^-8 * |O_ref|.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle.attention import attention_batch  # noqa: E402
from workloads import bf16_bits_to_f32  # noqa: E402
from workloads.attn import PAGE, make_attn_batch  # noqa: E402

from tests.gpu_util import to_dev  # noqa: E402


def _run(bs, b, poison_tail=False):
    kc, vc = b.k_cache.copy(), b.v_cache.copy()
    if poison_tail:  # cache slots past each context and unused pages hold NaN
        used = np.zeros(kc.shape[0], bool)
        for r in range(len(b.ctx_len)):
            L = int(b.ctx_len[r])
            npg = (L + PAGE - 1) // PAGE
            used[b.page_table[r, :npg]] = True
            last = b.page_table[r, npg - 1]
            kc[last, :, L - (npg - 1) * PAGE:] = 0x7FC0
            vc[last, :, L - (npg - 1) * PAGE:] = 0x7FC0
        kc[~used] = 0x7FC0
        vc[~used] = 0x7FC0
    q = to_dev(b.q.view(np.int16))
    out = bs.bs_unified_attention(q, to_dev(kc.view(np.int16)), to_dev(vc.view(np.int16)), to_dev(b.page_table),
                                  to_dev(b.ctx_len), b.ctx_len, list(np.diff(b.q_off)), b.H_kv)
    torch.cuda.synchronize()
    return bf16_bits_to_f32(out.cpu().numpy().view(np.uint16)).astype(np.float64)


def _check(b, got):
    ref = attention_batch(b)
    for r in range(len(b.ctx_len)):
        r0, r1 = int(b.q_off[r]), int(b.q_off[r + 1])
        from workloads.attn import logical_kv

        _, v = logical_kv(b, r)
        vmax = float(np.abs(bf16_bits_to_f32(v)).max())
        err = np.abs(got[r0:r1] - ref[r0:r1])
        bound = 2.0 ** -8 * vmax + 2.0 ** -8 * np.abs(ref[r0:r1])
        assert np.isfinite(got[r0:r1]).all(), r
        assert (err <= bound).all(), (r, float(err.max()), float((err - bound).max()))


@pytest.mark.parametrize("q_len,ctx,H_q,H_kv", [
    ([1, 5, 9], [70, 200, 130], 28, 4),                  # Qwen2.5-7B heads, ragged
    ([1, 1, 1, 1], [64, 128, 129, 1], 28, 4),            # decode only; page / tile edges; 1-token ctx
    ([9, 3, 1, 5, 2], [9, 300, 2100, 4097, 65], 32, 8),  # Qwen3-8B heads; 2+ KV splits
    ([4, 1], [5000, 4100], 16, 8),                       # G = 2
    ([32], [200], 4, 1),                                 # G = 4, 128 rows
    ([17, 1, 9], [300, 5000, 2049], 28, 4),              # k = 16 drafts (LC): 17 x 7 = 119 rows
])
def test_unified_attention_parity(bs, q_len, ctx, H_q, H_kv):
    b = make_attn_batch(len(ctx) * 7 + H_q, q_len, ctx, H_q=H_q, H_kv=H_kv)
    _check(b, _run(bs, b))


def test_unified_attention_ignores_cache_past_context(bs):
    """NaN in the cache past each request's context and in unused pages never reaches O (the
    kernel zeroes the V rows of masked keys; TMA zero-fills pages past the context)."""
    b = make_attn_batch(5, [1, 4, 9, 2], [77, 130, 191, 64 * 3 + 5], H_q=28, H_kv=4)
    _check(b, _run(bs, b, poison_tail=True))


def test_unified_equals_batch_split(bs):
    """Unified (one launch, mixed q_len) == the batch-split baseline (decode requests and
    speculative requests in separate launches): same rows, bit-identical (the work
    units of a request do not depend on the other requests)."""
    q_len, ctx = [1, 5, 1, 5, 1], [300, 260, 1000, 520, 77]
    b = make_attn_batch(8, q_len, ctx, H_q=28, H_kv=4)
    got = _run(bs, b)
    for sel in ([0, 2, 4], [1, 3]):
        from workloads.attn import AttnBatch

        qo = np.zeros(len(sel) + 1, np.int32)
        qo[1:] = np.cumsum([q_len[i] for i in sel])
        q = np.concatenate([b.q[b.q_off[i]:b.q_off[i + 1]] for i in sel])
        sub = AttnBatch(q=q, k_cache=b.k_cache, v_cache=b.v_cache, page_table=b.page_table[sel],
                        ctx_len=b.ctx_len[sel], q_off=qo, H_q=b.H_q, H_kv=b.H_kv, d=b.d)
        part = _run(bs, sub)
        rows = np.concatenate([np.arange(b.q_off[i], b.q_off[i + 1]) for i in sel])
        np.testing.assert_array_equal(part, got[rows])


def test_synth_attn_values_match_numpy(bs):
    from workloads.attn import _vals

    n = 100_003
    t = torch.empty(n, dtype=torch.int16, device="cuda")
    mult = float(np.float32(1.0 / 147.8))
    bs.bsx_synth_attn_values(t, (9 * 1000003 + 2) & 0xFFFFFFFF, mult)
    torch.cuda.synchronize()
    from workloads import f32_to_bf16_bits

    assert np.array_equal(t.cpu().numpy().view(np.uint16), f32_to_bf16_bits(_vals(9, 2, n, 1.0)))


def test_unified_attention_table2_full_size_sampled(bs):
    """At the size the bench times (the paper's Table 2 setting: 128 requests x 8192 keys, 32 of
    them with 4 drafts, Qwen2.5-7B heads, values from the device twin of the generator, shuffled
    pages): sampled requests (speculative and plain, first / last) against the oracle."""
    from oracle.attention import attention_request
    from workloads.attn import PAGE as PG

    H_q, H_kv, D, B, ctx_len = 28, 4, 128, 128, 8192
    rng = np.random.default_rng(0)
    q_len = np.ones(B, dtype=np.int32)
    spec = rng.choice(B, 32, replace=False)
    q_len[spec] = 5
    ctx = np.full(B, ctx_len, dtype=np.int32)
    npg = ctx_len // PG
    perm = np.random.default_rng(1).permutation(B * npg).astype(np.int32)
    pt = perm.reshape(B, npg)
    mult = float(np.float32(1.0 / 147.8))
    kc = torch.empty((B * npg, H_kv, PG, D), dtype=torch.int16, device="cuda")
    vc = torch.empty_like(kc)
    bs.bsx_synth_attn_values(kc, 11, mult)
    bs.bsx_synth_attn_values(vc, 12, mult)
    q = torch.empty((int(q_len.sum()), H_q, D), dtype=torch.int16, device="cuda")
    bs.bsx_synth_attn_values(q, 13, mult)
    out = bs.bs_unified_attention(q, kc, vc, to_dev(pt), to_dev(ctx), ctx, q_len, H_kv)
    torch.cuda.synchronize()
    q_off = np.concatenate([[0], np.cumsum(q_len)])
    sample = sorted({0, B - 1, int(spec[0]), int(spec[1]), int(np.setdiff1d(np.arange(B), spec)[3])})
    for b in sample:
        pages = torch.from_numpy(pt[b].astype(np.int64)).cuda()
        k = kc[pages].permute(0, 2, 1, 3).reshape(ctx_len, H_kv, D).cpu().numpy().view(np.uint16)
        v = vc[pages].permute(0, 2, 1, 3).reshape(ctx_len, H_kv, D).cpu().numpy().view(np.uint16)
        qb = q[q_off[b]:q_off[b + 1]].cpu().numpy().view(np.uint16)
        ref = attention_request(qb, k, v, H_kv)
        got = bf16_bits_to_f32(out[q_off[b]:q_off[b + 1]].cpu().numpy().view(np.uint16)).astype(np.float64)
        vmax = float(np.abs(bf16_bits_to_f32(v)).max())
        bound = 2.0 ** -8 * vmax + 2.0 ** -8 * np.abs(ref)
        assert (np.abs(got - ref) <= bound).all(), b
