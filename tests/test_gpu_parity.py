"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by element on
the same seeded inputs.  Bit-exact on drafts, accepted lengths, emitted tokens and the
integer normaliser Z; softmax normalisers within 1e-5 relative of the oracle's fp64 sum.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import TargetSpec, bank_rows, bf16_bits_to_f32, f32_to_bf16_bits  # noqa: E402

from tests.gpu_util import bank_numpy, pools_for, setup_rollouts, to_dev  # noqa: E402


def _verify_gpu(bs, ctx, rows_dense, drafts, dlen, k, T, top_p, stride=None, top_k=0):
    """Run bs_verify_step on dense rows [n, k+1, V] (uint16) with rollouts already begun."""
    n = drafts.shape[0]
    V = rows_dense.shape[2]
    stride = stride or V
    if stride != V:
        buf = np.zeros((n, k + 1, stride), dtype=np.uint16)
        buf[:, :, :V] = rows_dense
    else:
        buf = rows_dense
    lg = to_dev(buf.view(np.int16).reshape(-1))
    slots = to_dev(np.arange(n, dtype=np.int32))
    out_t = torch.full((n, k + 1), -7, dtype=torch.int32, device="cuda")
    out_l = torch.zeros(n, dtype=torch.int32, device="cuda")
    out_a = torch.zeros(n, dtype=torch.int32, device="cuda")
    out_n = torch.zeros((n, k + 1), dtype=torch.float32, device="cuda")
    out_z = torch.zeros((n, k + 1), dtype=torch.int64, device="cuda")
    ctx.bs_verify_step(slots, lg, None, stride, to_dev(drafts.astype(np.int32)),
                       to_dev(dlen.astype(np.int32)), k, T, top_p, out_t, out_l, out_a, out_n, out_z,
                       top_k=top_k)
    torch.cuda.synchronize()
    return (out_t.cpu().numpy(), out_l.cpu().numpy(), out_a.cpu().numpy(), out_n.cpu().numpy(),
            out_z.cpu().numpy().view(np.uint64))


def _begin(bs, ctx, n, pos_max_len, uids, M):
    slots = to_dev(np.arange(n, dtype=np.int32))
    tail = np.full((n, M), -1, dtype=np.int32)
    tail[:, -1] = 0
    ctx.bs_rollout_begin(slots, to_dev(np.asarray(uids, dtype=np.uint64).view(np.int64)),
                         to_dev(np.zeros(n, dtype=np.int32)), to_dev(tail),
                         to_dev(np.asarray(pos_max_len, dtype=np.int32)))


def _compare_step(orc, rows, drafts, dlen, k, T, top_p, seed, uids, max_len, eos, got,
                  pos=0, top_k=0):
    ot, ol, oa, on, oz = got
    for b in range(drafts.shape[0]):
        q = int(dlen[b])
        o = orc.verify_one([rows[b, j] for j in range(k + 1)], T, top_p, seed, int(uids[b]), pos,
                           int(max_len[b]), eos, False, [int(x) for x in drafts[b, :q]], k, top_k=top_k)
        assert int(ol[b]) == len(o.tokens), (b, ol[b], o.tokens)
        assert [int(x) for x in ot[b, : ol[b]]] == o.tokens, (b, ot[b], o.tokens)
        assert int(oa[b]) == o.accepted
        for j in range(o.rows_used):
            assert int(oz[b, j]) == o.z[j], (b, j)
            if T > 0:
                assert abs(float(on[b, j]) / o.norm_fp64[j] - 1) < 1e-5, (b, j)
        for j in range(o.rows_used, k + 1):
            assert int(oz[b, j]) == 0 and float(on[b, j]) == 0.0


KERNELS = ["rows", "cluster"]  # bsx_set_verify_kernel: every verify kernel


@pytest.mark.parametrize("path", KERNELS)
@pytest.mark.parametrize("V,T,stride", [(1024, 1.0, None), (1000, 0.7, None), (4096, 1.3, None),
                                        (1001, 1.0, 1003), (1024, 0.0, None), (33, 1.0, None),
                                        (151936, 1.0, None), (151936, 0.0, None),
                                        (200003, 0.9, None)])
def test_verify_step_parity(bs, orc, V, T, stride, path):
    """Random logits rows (several tiles + ragged tail, odd strides), random drafts mixing
    the argmax (often accepted) with random tokens."""
    rng = np.random.default_rng(V + int(T * 10))
    k = 4 if V < 100000 else 8
    n = 48 if V < 100000 else 12
    rows = f32_to_bf16_bits(rng.normal(0, 2.0, size=(n, k + 1, V)).astype(np.float32))
    # make some rows peaked so acceptance happens
    for b in range(n):
        for j in range(k + 1):
            if rng.random() < 0.6:
                rows[b, j, rng.integers(0, V)] = f32_to_bf16_bits(np.float32(9.0))
    argm = bf16_bits_to_f32(rows).argmax(axis=2)
    drafts = np.where(rng.random((n, k)) < 0.7, argm[:, :k], rng.integers(0, V, (n, k)))
    dlen = rng.integers(0, k + 1, n)
    max_len = np.where(rng.random(n) < 0.2, rng.integers(1, 4, n), 1000)
    seed = 0xABCDEF
    ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=8, max_rollouts=n,
                     pool_capacity_tokens=16, pool_capacity_seqs=4, seed=seed)
    ctx.bsx_set_verify_kernel(path)
    uids = np.arange(n, dtype=np.uint64) * np.uint64(7919) + np.uint64(3)
    _begin(bs, ctx, n, max_len, uids, 8)
    got = _verify_gpu(bs, ctx, rows, drafts, dlen, k, T, 1.0, stride)
    assert ctx.bs_sync_status() == 0
    _compare_step(orc, rows, drafts, dlen, k, T, 1.0, seed, uids, max_len, -1, got)


def _topp_rows(rng, kind, n, k, V):
    if kind == "quant":      # logits on a 0.5 grid: large tie groups straddle the threshold
        vals = np.round(rng.normal(0, 2.0, size=(n, k + 1, V)) * 2) / 2
    elif kind == "dense0":   # logits near 0, where distinct bf16 keys share one mass
        vals = rng.uniform(-0.01, 0.01, size=(n, k + 1, V))
    else:
        vals = rng.normal(0, 2.0, size=(n, k + 1, V))
    rows = f32_to_bf16_bits(vals.astype(np.float32))
    for b in range(n):
        for j in range(k + 1):
            if rng.random() < 0.5:
                rows[b, j, rng.integers(0, V, 3)] = f32_to_bf16_bits(np.float32(3.0))
    return rows


@pytest.mark.parametrize("V,T,top_p,kind,stride", [
    (1024, 1.0, 0.9, "normal", None), (4099, 0.7, 0.5, "normal", None),
    (1000, 1.3, 0.999, "quant", None), (4096, 1.0, 0.3, "quant", None),
    (3000, 1.0, 0.6, "dense0", None), (1001, 1.0, 0.8, "quant", 1003),
    (513, 1.0, 1e-6, "normal", None), (151936, 1.0, 0.95, "normal", None),
    (151936, 0.8, 0.7, "dense0", None),
    # a slice too large to stage in shared memory beside the histograms: the passes stream L2
    (300001, 1.0, 0.9, "normal", None)])
def test_verify_top_p_parity(bs, orc, V, T, top_p, kind, stride):
    """Top-p (reading R5, tie-closed nucleus): the mass-weighted key select on the GPU keeps
    exactly the oracle's set; accepted lengths, tokens and Z' bit-exact."""
    rng = np.random.default_rng(V * 7 + int(top_p * 1000))
    k = 4 if V < 100000 else 6
    n = 40 if V < 100000 else 8
    rows = _topp_rows(rng, kind, n, k, V)
    argm = bf16_bits_to_f32(rows).argmax(axis=2)
    drafts = np.where(rng.random((n, k)) < 0.7, argm[:, :k], rng.integers(0, V, (n, k)))
    dlen = rng.integers(0, k + 1, n)
    max_len = np.full(n, 1000)
    seed = 0x5EED
    ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=8, max_rollouts=n,
                     pool_capacity_tokens=16, pool_capacity_seqs=4, seed=seed)
    uids = np.arange(n, dtype=np.uint64) * np.uint64(104729) + np.uint64(5)
    _begin(bs, ctx, n, max_len, uids, 8)
    got = _verify_gpu(bs, ctx, rows, drafts, dlen, k, T, top_p, stride)
    assert ctx.bs_sync_status() == 0
    _compare_step(orc, rows, drafts, dlen, k, T, top_p, seed, uids, max_len, -1, got)


@pytest.mark.parametrize("V,T,top_p,top_k,kind", [
    (1024, 1.0, 1.0, 1, "normal"), (1024, 1.0, 1.0, 50, "normal"), (4099, 0.7, 1.0, 7, "quant"),
    (1000, 1.0, 1.0, 3, "dense0"), (3000, 1.3, 0.9, 20, "normal"), (4096, 1.0, 0.5, 200, "quant"),
    (1001, 1.0, 0.8, 2, "quant"), (2048, 1.0, 1.0, 2047, "normal"), (2048, 1.0, 1.0, 4096, "normal"),
    (151936, 1.0, 1.0, 50, "normal"), (151936, 1.0, 0.95, 40, "dense0"), (300001, 1.0, 0.95, 30, "quant")])
def test_verify_top_k_parity(bs, orc, V, T, top_p, top_k, kind):
    """Top-k then top-p (readings R5k, R5; SPEC S:74 order): the count-weighted key select on
    the GPU keeps exactly the oracle's tie-closed top-k set, top-p then runs on it; accepted
    lengths, tokens and Z' bit-exact ("quant" rows have many tied logits at the k-th place)."""
    rng = np.random.default_rng(V * 11 + top_k)
    k = 4 if V < 100000 else 6
    n = 40 if V < 100000 else 8
    rows = _topp_rows(rng, kind, n, k, V)
    argm = bf16_bits_to_f32(rows).argmax(axis=2)
    drafts = np.where(rng.random((n, k)) < 0.7, argm[:, :k], rng.integers(0, V, (n, k)))
    dlen = rng.integers(0, k + 1, n)
    max_len = np.full(n, 1000)
    seed = 0x5EED
    ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=8, max_rollouts=n,
                     pool_capacity_tokens=16, pool_capacity_seqs=4, seed=seed)
    uids = np.arange(n, dtype=np.uint64) * np.uint64(7919) + np.uint64(3)
    _begin(bs, ctx, n, max_len, uids, 8)
    got = _verify_gpu(bs, ctx, rows, drafts, dlen, k, T, top_p, top_k=top_k)
    assert ctx.bs_sync_status() == 0
    _compare_step(orc, rows, drafts, dlen, k, T, top_p, seed, uids, max_len, -1, got, top_k=top_k)


@pytest.mark.parametrize("path", KERNELS)
def test_verify_eos_and_edge_cases(bs, orc, path):
    """Accepted EOS ends the block; q=0 is a plain sample; -inf logits; max_len clamp."""
    V, k, n, eos = 64, 4, 32, 5
    rng = np.random.default_rng(1)
    vals = rng.normal(0, 1, (n, k + 1, V)).astype(np.float32)
    vals[:, :, 7] = -np.inf
    vals[::2, 1, eos] = 12.0  # EOS very likely at row 1
    rows = f32_to_bf16_bits(vals)
    drafts = rng.integers(0, V, (n, k))
    drafts[:, 1] = eos
    drafts[::3, 0] = 7  # zero-mass draft token: rejected at row 0
    dlen = np.full(n, k)
    dlen[::5] = 0
    max_len = np.full(n, 100)
    max_len[::7] = 2
    seed = 99
    ctx = bs.Context(vocab=V, eos_id=eos, k_max=k, match_max=8, max_rollouts=n,
                     pool_capacity_tokens=16, pool_capacity_seqs=4, seed=seed)
    ctx.bsx_set_verify_kernel(path)
    uids = np.arange(n, dtype=np.uint64) + np.uint64(11)
    _begin(bs, ctx, n, max_len, uids, 8)
    got = _verify_gpu(bs, ctx, rows, drafts, dlen, k, 1.0, 1.0)
    assert ctx.bs_sync_status() == 0
    _compare_step(orc, rows, drafts, dlen, k, 1.0, 1.0, seed, uids, max_len, eos, got)


@pytest.mark.parametrize("path", KERNELS)
def test_verify_device_errors(bs, path):
    V, k, n = 64, 2, 4
    rows = np.zeros((n, k + 1, V), dtype=np.uint16)
    rows[1, 0, 3] = 0x7FC0  # NaN
    ctx = bs.Context(vocab=V, k_max=k, match_max=8, max_rollouts=n, pool_capacity_tokens=16,
                     pool_capacity_seqs=4)
    ctx.bsx_set_verify_kernel(path)
    _begin(bs, ctx, n, [10] * n, np.arange(n, dtype=np.uint64), 8)
    _verify_gpu(bs, ctx, rows, np.zeros((n, k), np.int64), np.full(n, 2), k, 1.0, 1.0)
    assert ctx.bs_sync_status() & 0x1
    _verify_gpu(bs, ctx, np.zeros((n, k + 1, V), np.uint16), np.full((n, k), V + 3),
                np.full(n, 2), k, 1.0, 1.0)
    assert ctx.bs_sync_status() & 0x8
    allneg = np.full((n, k + 1, V), 0xFF80, dtype=np.uint16)
    _verify_gpu(bs, ctx, allneg, np.zeros((n, k), np.int64), np.full(n, 1), k, 1.0, 1.0)
    assert ctx.bs_sync_status() & 0x2


def _error_rows(V, k, seed=5):
    """Four rollouts (k = 2) around invalid rows (reading R0): 0 rejects d_1 for certain
    (mass(d_1) = 0, R7) so its NaN row 1 is never needed; 1 has a NaN in row 0 (needed);
    2 accepts d_1 for certain (p(d_1) = 1) and has a NaN in row 1 (needed); 3 is ordinary."""
    n = 4
    rows = bank_rows(seed, np.arange(n * (k + 1)), V, 6.0).reshape(n, k + 1, V).copy()
    drafts = np.tile(np.arange(1, k + 1), (n, 1)).astype(np.int64)
    rows[0, 0, drafts[0, 0]] = 0xFF80  # -inf: p(d_1) = 0
    rows[0, 1, 7] = 0x7FC0             # NaN in a row Alg. 1 never reads
    rows[1, 0, 9] = 0x7FC0             # NaN in row 0: needed
    rows[2, 0, :] = 0xFF80
    rows[2, 0, drafts[2, 0]] = 0x3F80  # only d_1 finite: p(d_1) = 1
    rows[2, 1, 11] = 0x7F80            # +inf in row 1: needed
    return rows, drafts, np.full(n, k)


@pytest.mark.parametrize("path", KERNELS)
@pytest.mark.parametrize("V", [64, 4099])
def test_verify_error_only_if_needed(bs, orc, path, V):
    """The error word reports an invalid row only if Alg. 1 reads it (the oracle stops there,
    P:538-561 read in order); a rollout whose needed row is invalid emits nothing and the
    commit stops it; the other rollouts match the oracle token for token."""
    k, n, seed = 2, 4, 3
    rows, drafts, dlen = _error_rows(V, k)
    uids = np.arange(n, dtype=np.uint64) + np.uint64(5)
    ml = np.full(n, 50)
    for case in ("unneeded_only", "needed"):
        r = rows.copy()
        if case == "unneeded_only":  # rollouts 1 and 2 made valid again
            r[1, 0, 9] = 0
            r[2, 1, 11] = 0
        ctx = bs.Context(vocab=V, k_max=k, match_max=8, max_rollouts=n, pool_capacity_tokens=16,
                         pool_capacity_seqs=4, seed=seed)
        ctx.bsx_set_verify_kernel(path)
        _begin(bs, ctx, n, ml, uids, 8)
        ot, ol, oa, _, _ = _verify_gpu(bs, ctx, r, drafts, dlen, k, 1.0, 1.0)
        word = ctx.bs_sync_status()
        bad = {1, 2} if case == "needed" else set()
        assert (word & 0x1 != 0) == bool(bad), (case, word)
        for b in range(n):
            if b in bad:
                with pytest.raises(orc.OracleError):
                    orc.verify_one([r[b, j] for j in range(k + 1)], 1.0, 1.0, seed, int(uids[b]), 0,
                                   int(ml[b]), -1, False, [int(x) for x in drafts[b]], k)
                assert ol[b] == 0 and oa[b] == 0 and (ot[b] == -1).all()
                continue
            o = orc.verify_one([r[b, j] for j in range(k + 1)], 1.0, 1.0, seed, int(uids[b]), 0,
                               int(ml[b]), -1, False, [int(x) for x in drafts[b]], k)
            assert [int(x) for x in ot[b, : ol[b]]] == o.tokens, (case, b)
        # the commit stops a rollout whose step emitted nothing (an error stop)
        slots = to_dev(np.arange(n, dtype=np.int32))
        fin = torch.zeros(n, dtype=torch.int32, device="cuda")
        ctx.bs_commit(slots, to_dev(ot.astype(np.int32)), to_dev(ol.astype(np.int32)), k, fin)
        torch.cuda.synchronize()
        assert [int(x) for x in fin.cpu()] == [1 if b in bad else 0 for b in range(n)]


# ------------------------------------------------------------------ lookup
def _gpu_lookup(bs, ctx, seq_prompt, seq_off, tokens, ctxs, prompt_of, k, M, max_len=1 << 20,
                rl_step=1, ngram=None, min_token_prob=None):
    n = len(ctxs)
    if min_token_prob is not None:
        ctx.bs_draft_set_min_token_prob(min_token_prob)  # applies from the seal below (C1)
    ctx.bs_draft_pool_put(rl_step, to_dev(seq_prompt.astype(np.int32)), to_dev(seq_off),
                          to_dev(tokens.astype(np.int32)) if len(tokens) else
                          to_dev(np.zeros(1, np.int32)), int(len(tokens)))
    ctx.bs_draft_pool_seal(rl_step)
    tail = np.full((n, M), -1, dtype=np.int32)
    for b, c in enumerate(ctxs):
        c = list(c)[-M:]
        tail[b, M - len(c):] = c
    slots = to_dev(np.arange(n, dtype=np.int32))
    ctx.bs_rollout_begin(slots, to_dev(np.arange(n, dtype=np.int64)),
                         to_dev(np.asarray(prompt_of, dtype=np.int32)), to_dev(tail),
                         to_dev(np.full(n, max_len, dtype=np.int32)))
    d = torch.zeros((n, k), dtype=torch.int32, device="cuda")
    dl = torch.zeros(n, dtype=torch.int32, device="cuda")
    ml = torch.zeros(n, dtype=torch.int32, device="cuda")
    if ngram is None:
        ctx.bs_draft_lookup(rl_step, slots, k, d, dl, ml)
    else:
        ctx.bs_draft_lookup_ngram(rl_step, slots, k, ngram[0], ngram[1], d, dl, ml)
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    return d.cpu().numpy(), dl.cpu().numpy(), ml.cpu().numpy()


@pytest.mark.parametrize("vocab,n_min,n_max,M,k", [(3, 1, 8, 8, 4), (5, 2, 6, 8, 3), (2, 1, 32, 32, 16),
                                                   (50, 1, 4, 16, 8), (4, 3, 3, 8, 5)])
def test_ngram_lookup_parity_random_pools(bs, orc, vocab, n_min, n_max, M, k):
    """Draft-source variant f4 (reading N1): the GPU n-gram linear scan == the oracle's
    (drafts and match length n), random pools of several prompts, ragged and empty sequences,
    contexts copied from pool sequences (long matches), max_len clamps."""
    rng = np.random.default_rng(vocab * 31 + n_max)
    n_prompts = 5
    seqs, sp = [], []
    for P in range(n_prompts):
        for _ in range(int(rng.integers(0, 6))):
            seqs.append(rng.integers(0, vocab, int(rng.integers(0, 300))).astype(np.int32))
            sp.append(P)
    off = np.zeros(len(seqs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(s) for s in seqs])
    tokens = np.concatenate(seqs) if seqs and off[-1] else np.zeros(0, np.int32)
    ctxs, pof = [], []
    for _ in range(150):
        P = int(rng.integers(0, n_prompts))
        own = [s for s, p in zip(seqs, sp) if p == P and len(s) > 3]
        if own and rng.random() < 0.6:
            s = own[int(rng.integers(0, len(own)))]
            e = int(rng.integers(1, len(s) + 1))
            c = list(rng.integers(0, vocab, int(rng.integers(0, 5)))) + list(s[:e])
        else:
            c = list(rng.integers(0, vocab, int(rng.integers(1, 40))))
        ctxs.append([int(x) for x in c] or [0])
        pof.append(P)
    ctx = bs.Context(vocab=vocab, k_max=k, match_max=M, max_rollouts=len(ctxs),
                     pool_capacity_tokens=max(1, len(tokens)), pool_capacity_seqs=max(1, len(seqs)))
    max_len = 3 if vocab == 4 else 1 << 20
    d, dl, ml = _gpu_lookup(bs, ctx, np.asarray(sp), off, tokens, ctxs, pof, k, M, max_len=max_len,
                            ngram=(n_min, n_max))
    pools = {}
    for s_, p_ in zip(seqs, sp):
        pools.setdefault(p_, []).append([int(x) for x in s_])
    for b, (c, P) in enumerate(zip(ctxs, pof)):
        want, n = orc.lookup_ngram(pools.get(P, []), c[-M:], n_min, n_max, k)
        want = want[:max(0, max_len - 1)]  # L6 clamp at pos 0
        assert int(dl[b]) == len(want), (b, c, want, d[b], dl[b])
        assert [int(x) for x in d[b, :dl[b]]] == want, b
        assert int(ml[b]) == n, b


@pytest.mark.parametrize("vocab,Lmin,M,k,tau", [(3, 1, 8, 4, 0.0), (5, 1, 6, 3, 0.0), (4, 2, 8, 5, 0.0),
                                                (50, 1, 32, 8, 0.0), (2, 1, 32, 16, 0.0),
                                                (3, 1, 8, 4, 0.3), (4, 2, 8, 5, 0.5), (2, 1, 32, 16, 0.6),
                                                (5, 1, 6, 3, 1.0), (50, 1, 32, 8, 0.34)])
def test_lookup_parity_random_pools(bs, orc, vocab, Lmin, M, k, tau):
    """random pools x prefixes, GPU index lookup == brute-force oracle (drafts and
    anchor length), several prompts per pool; tau > 0: confidence-scored drafts (reading C1,
    the threshold applied by the index build, the oracle's descent stops at the same step)."""
    rng = np.random.default_rng(vocab * 100 + M)
    n_prompts = 6
    seqs, sp = [], []
    for P in range(n_prompts):
        for _ in range(int(rng.integers(0, 6))):
            L = int(rng.integers(0, 40))
            seqs.append(rng.integers(0, vocab, L).astype(np.int32))
            sp.append(P)
    off = np.zeros(len(seqs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(s) for s in seqs])
    tokens = np.concatenate(seqs) if seqs and off[-1] else np.zeros(0, np.int32)
    ctxs, pof = [], []
    for _ in range(200):
        P = int(rng.integers(0, n_prompts))
        # contexts: either random or copied from a pool sequence (long matches)
        own = [s for s, p in zip(seqs, sp) if p == P and len(s) > 3]
        if own and rng.random() < 0.6:
            s = own[int(rng.integers(0, len(own)))]
            e = int(rng.integers(1, len(s) + 1))
            c = list(rng.integers(0, vocab, int(rng.integers(0, 5)))) + list(s[:e])
        else:
            c = list(rng.integers(0, vocab, int(rng.integers(1, 40))))
        ctxs.append([int(x) for x in c] or [0])
        pof.append(P)
    ctx = bs.Context(vocab=vocab, k_max=k, match_max=M, match_min=Lmin, max_rollouts=len(ctxs),
                     pool_capacity_tokens=max(1, len(tokens)), pool_capacity_seqs=max(1, len(seqs)))
    d, dl, ml = _gpu_lookup(bs, ctx, np.asarray(sp, np.int32), off, tokens, ctxs, pof, k, M,
                            min_token_prob=tau if tau else None)
    pools = {}
    for s, P in zip(seqs, sp):
        pools.setdefault(P, []).append([int(x) for x in s])
    for b, c in enumerate(ctxs):
        want_d, want_m = orc.lookup(pools.get(pof[b], []), c[-M:], M, Lmin, k, tau)
        assert list(d[b, : dl[b]]) == want_d, (b, c, want_d, d[b], dl[b])
        assert int(ml[b]) == want_m, (b, c, ml[b], want_m)


def test_lookup_stale_and_clamp(bs, orc):
    V, k, M = 10, 4, 8
    seqs = [np.array([1, 2, 3, 4, 5, 6], np.int32)]
    off = np.array([0, 6], np.int64)
    ctx = bs.Context(vocab=V, k_max=k, match_max=M, max_rollouts=2, pool_capacity_tokens=16,
                     pool_capacity_seqs=2)
    d, dl, ml = _gpu_lookup(bs, ctx, np.array([0], np.int32), off, seqs[0], [[1, 2], [1, 2]],
                            [0, 0], k, M, max_len=3)
    assert list(dl) == [2, 2] and list(d[0, :2]) == [3, 4]  # clamp: max_len - pos - 1 = 2
    with pytest.raises(bs.BubbleSpecError):
        slots = to_dev(np.arange(2, dtype=np.int32))
        z = torch.zeros((2, k), dtype=torch.int32, device="cuda")
        ctx.bs_draft_lookup(2, slots, k, z, z[:, 0].contiguous())


@pytest.mark.parametrize("tau", [0.0, 0.9])  # 0.9: shortens 688 -> 534 drafted tokens here
def test_lookup_index_on_perturbed_pools(bs, orc, tau):
    """Qwen-shaped vocab, pools = 16 perturbed copies of a reference text (the bench's
    recipe): GPU == oracle on contexts sampled along the reference (tau > 0:
    confidence-scored drafts, reading C1)."""
    spec = TargetSpec(V=151936, nbank=64, mode="position")
    M, k = 32, 8
    prompts, tails, *_ = setup_rollouts(spec, 3, 1, M, 100)
    rng = np.random.default_rng(3)
    lens = rng.integers(50, 400, (3, 16))
    sp, off, tok = pools_for(spec, prompts, tails, 16, lens, 0.8, prefix=M)
    ctxs, pof = [], []
    for i, P in enumerate(prompts):
        s = tok[off[16 * i]: off[16 * i + 1]]
        for _ in range(40):
            e = int(rng.integers(1, len(s)))
            c = [int(x) for x in s[max(0, e - 40): e]]
            if rng.random() < 0.3:
                c[-1] = int(rng.integers(0, spec.V))
            ctxs.append(c)
            pof.append(int(P))
    ctx = bs.Context(vocab=spec.V, k_max=k, match_max=M, max_rollouts=len(ctxs),
                     pool_capacity_tokens=len(tok), pool_capacity_seqs=len(sp))
    d, dl, ml = _gpu_lookup(bs, ctx, sp, off, tok, ctxs, pof, k, M, min_token_prob=tau)
    pools = {}
    for s_i, P in enumerate(sp):
        pools.setdefault(int(P), []).append([int(x) for x in tok[off[s_i]:off[s_i + 1]]])
    if tau:  # the threshold must actually shorten some drafts on this workload
        plain = [len(orc.lookup(pools[pof[b]], c[-M:], M, 1, k)[0]) for b, c in enumerate(ctxs)]
        assert sum(plain) > int(dl.sum())
    for b, c in enumerate(ctxs):
        want_d, want_m = orc.lookup(pools[pof[b]], c[-M:], M, 1, k, tau)
        assert list(d[b, : dl[b]]) == want_d and int(ml[b]) == want_m, b


# ------------------------------------------------------------------ synthetic twins
def test_synth_bank_matches_numpy(bs):
    V, rows = 151936, 6
    bank = torch.empty((rows, V), dtype=torch.int16, device="cuda")
    bs.bsx_synth_bank(bank, rows, V, 1234, 11.5)
    torch.cuda.synchronize()
    want = bank_rows(1234, np.arange(rows), V, 11.5)
    assert np.array_equal(bank.cpu().numpy().view(np.uint16), want)


def _random_step(rng, n, k, V, peaked=0.6):
    rows = f32_to_bf16_bits(rng.normal(0, 2.0, size=(n, k + 1, V)).astype(np.float32))
    for b in range(n):
        for j in range(k + 1):
            if rng.random() < peaked:
                rows[b, j, rng.integers(0, V)] = f32_to_bf16_bits(np.float32(9.0))
    argm = bf16_bits_to_f32(rows).argmax(axis=2)
    drafts = np.where(rng.random((n, k)) < 0.8, argm[:, :k], rng.integers(0, V, (n, k)))
    dlen = rng.integers(0, k + 1, n)
    return rows, drafts, dlen


@pytest.mark.parametrize("eager", [True, False])
@pytest.mark.parametrize("n_live,n", [(1, 64), (4, 64), (30, 64), (64, 64)])
def test_cluster_scheduler_mostly_finished(bs, orc, monkeypatch, eager, n_live, n):
    """The cluster kernel's scheduler (in-kernel plan, compacted live list, eager all-rows
    mode for small live batches vs lazy ready/static/speculative claims): most slots
    finished (max_len = 0) must emit nothing; live ones match the oracle bit for bit, and the
    result does not depend on the scheduling mode."""
    if not eager:
        monkeypatch.setenv("BS_NO_EAGER", "1")
    rng = np.random.default_rng(7 * n_live + n)
    V, k = 4099, 6
    rows, drafts, dlen = _random_step(rng, n, k, V)
    live = rng.permutation(n)[:n_live]
    max_len = np.zeros(n, dtype=np.int64)
    max_len[live] = 1000
    seed = 0x1234
    ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=8, max_rollouts=n,
                     pool_capacity_tokens=16, pool_capacity_seqs=4, seed=seed)
    ctx.bsx_set_verify_kernel("cluster")
    uids = np.arange(n, dtype=np.uint64) * np.uint64(104729) + np.uint64(11)
    _begin(bs, ctx, n, max_len, uids, 8)
    got = _verify_gpu(bs, ctx, rows, drafts, dlen, k, 1.0, 1.0)
    assert ctx.bs_sync_status() == 0
    ot, ol, oa, on, oz = got
    dead = np.setdiff1d(np.arange(n), live)
    assert (ol[dead] == 0).all() and (ot[dead] == -1).all()
    sel = np.sort(live)
    _compare_step(orc, rows[sel], drafts[sel], dlen[sel], k, 1.0, 1.0, seed, uids[sel], max_len[sel], -1,
                  tuple(x[sel] for x in got))


def test_cluster_scheduler_repeated_launches(bs, orc):
    """Many launches on one context (the scheduler's per-launch epoch, counter resets by the
    last CTA out, plan records overwritten each launch) with a changing live set."""
    rng = np.random.default_rng(99)
    V, k, n = 2048, 4, 40
    seed = 0x77
    ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=8, max_rollouts=n,
                     pool_capacity_tokens=16, pool_capacity_seqs=4, seed=seed)
    ctx.bsx_set_verify_kernel("cluster")
    uids = np.arange(n, dtype=np.uint64) + np.uint64(5)
    for it in range(12):
        max_len = np.where(rng.random(n) < 0.5, 1000, 0)
        _begin(bs, ctx, n, max_len, uids, 8)
        rows, drafts, dlen = _random_step(rng, n, k, V)
        got = _verify_gpu(bs, ctx, rows, drafts, dlen, k, 1.0 if it % 3 else 0.0, 1.0)
        assert ctx.bs_sync_status() == 0
        live = np.nonzero(max_len)[0]
        _compare_step(orc, rows[live], drafts[live], dlen[live], k, 1.0 if it % 3 else 0.0, 1.0, seed,
                      uids[live], max_len[live], -1, tuple(x[live] for x in got))


@pytest.mark.parametrize("k", [2, 4, 8, 16])
def test_acceptance_sweep_k_qwen_vocab(bs, orc, k):
    """SWEEP config shapes (BASELINE.json configs[4]): k in {2, 4, 8, 16} at V = 151936 through
    the default (cluster) kernel, drafts mixing the argmax with random tokens."""
    rng = np.random.default_rng(1000 + k)
    V, n = 151936, 6
    rows, drafts, dlen = _random_step(rng, n, k, V, peaked=0.7)
    dlen[:] = k
    max_len = np.full(n, 100000)
    seed = 0xC0FFEE
    ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=32, max_rollouts=n,
                     pool_capacity_tokens=16, pool_capacity_seqs=4, seed=seed)
    uids = np.arange(n, dtype=np.uint64) + np.uint64(1 << 33)
    _begin(bs, ctx, n, max_len, uids, 32)
    got = _verify_gpu(bs, ctx, rows, drafts, dlen, k, 1.0, 1.0)
    assert ctx.bs_sync_status() == 0
    _compare_step(orc, rows, drafts, dlen, k, 1.0, 1.0, seed, uids, max_len, -1, got)


def test_long_context_config_topp(bs, orc):
    """LC config shapes (BASELINE.json configs[2]): V = 151936, k = 16, top-p 0.95, T = 1
    (the top-p kernel), with max_len clamping two of the drafts (reading L6)."""
    rng = np.random.default_rng(4242)
    V, n, k = 151936, 4, 16
    rows, drafts, dlen = _random_step(rng, n, k, V, peaked=0.7)
    dlen[:] = k
    max_len = np.array([32768, 32768, 9, 3])  # the last two clamp q (reading L6)
    seed = 0xFEED
    ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=32, max_rollouts=n,
                     pool_capacity_tokens=16, pool_capacity_seqs=4, seed=seed)
    uids = np.arange(n, dtype=np.uint64) + np.uint64(77)
    _begin(bs, ctx, n, max_len, uids, 32)
    got = _verify_gpu(bs, ctx, rows, drafts, dlen, k, 1.0, 0.95)
    assert ctx.bs_sync_status() == 0
    _compare_step(orc, rows, drafts, dlen, k, 1.0, 0.95, seed, uids, max_len, -1, got)


def test_back_to_back_verify_calls(bs, orc):
    """Several bs_verify_step calls enqueued back to back on one stream (no synchronisation,
    no kernel in between): the cluster kernel plans before griddepcontrol.wait, which is only
    safe because every verify launch releases its dependents at exit.  Each call has its own
    inputs and outputs; each must match the oracle."""
    rng = np.random.default_rng(31337)
    V, k, n, calls = 4096, 6, 24, 6
    seed = 0x51DE
    ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=8, max_rollouts=n,
                     pool_capacity_tokens=16, pool_capacity_seqs=4, seed=seed)
    uids = np.arange(n, dtype=np.uint64) + np.uint64(900)
    max_len = np.full(n, 1000)
    _begin(bs, ctx, n, max_len, uids, 8)
    torch.cuda.synchronize()
    slots = to_dev(np.arange(n, dtype=np.int32))
    ins, outs = [], []
    for c in range(calls):
        rows, drafts, dlen = _random_step(rng, n, k, V)
        lg = to_dev(rows.view(np.int16).reshape(-1))
        dr, dl = to_dev(drafts.astype(np.int32)), to_dev(dlen.astype(np.int32))
        o = (torch.full((n, k + 1), -7, dtype=torch.int32, device="cuda"),
             torch.zeros(n, dtype=torch.int32, device="cuda"), torch.zeros(n, dtype=torch.int32, device="cuda"),
             torch.zeros((n, k + 1), dtype=torch.float32, device="cuda"),
             torch.zeros((n, k + 1), dtype=torch.int64, device="cuda"))
        ins.append((rows, drafts, dlen, lg, dr, dl))
        outs.append(o)
    torch.cuda.synchronize()
    for c in range(calls):  # enqueue all, then synchronise once
        rows, drafts, dlen, lg, dr, dl = ins[c]
        ot, ol, oa, on, oz = outs[c]
        ctx.bs_verify_step(slots, lg, None, V, dr, dl, k, 1.0 if c % 2 else 0.8, 1.0, ot, ol, oa, on, oz)
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    for c in range(calls):
        rows, drafts, dlen = ins[c][:3]
        got = (outs[c][0].cpu().numpy(), outs[c][1].cpu().numpy(), outs[c][2].cpu().numpy(),
               outs[c][3].cpu().numpy(), outs[c][4].cpu().numpy().view(np.uint64))
        _compare_step(orc, rows, drafts, dlen, k, 1.0 if c % 2 else 0.8, 1.0, seed, uids, max_len, -1, got)
