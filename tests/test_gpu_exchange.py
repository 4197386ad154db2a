"""Cross-rank draft exchange ("each rollout DP rank builds and
maintains suffix indices only for the prompts it is responsible for", "dispatch
pre-generated draft responses to each rollout rank according to their assigned prompts") on
the GPU through the C-ABI: bs_nccl_unique_id -> bs_nccl_comm_init -> bs_draft_pool_put ->
bs_draft_exchange (NCCL all-gather + device gather) -> bs_draft_pool_seal -> bs_draft_lookup,
compared with the brute-force oracle lookup over the pools the rank owns."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.gpu_util import to_dev  # noqa: E402


def _random_pools(seed, n_prompts, vocab, prompt_base=0):
    rng = np.random.default_rng(seed)
    seqs, sp = [], []
    for P in range(n_prompts):
        for _ in range(int(rng.integers(1, 6))):
            seqs.append(rng.integers(0, vocab, int(rng.integers(1, 60))).astype(np.int32))
            sp.append(prompt_base + P)
    off = np.zeros(len(seqs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(s) for s in seqs])
    return np.asarray(sp, np.int32), off, np.concatenate(seqs)


def _lookup_vs_oracle(bs, orc, ctx, rl_step, pools_np, prompts, vocab, k, M, seed):
    """Lookups of random contexts of the given prompts vs the oracle over pools_np."""
    from oracle.rollout import pools_by_prompt

    rng = np.random.default_rng(seed)
    pools = pools_by_prompt(*pools_np)
    ctxs, pof = [], []
    for _ in range(128):
        P = int(rng.choice(prompts))
        src = pools.get(P, [[0]])
        s = src[int(rng.integers(0, len(src)))]
        a = int(rng.integers(0, len(s)))
        c = list(s[max(0, a - int(rng.integers(1, 20))): a + 1])
        if rng.random() < 0.3:
            c = c + [int(rng.integers(0, vocab))]
        ctxs.append(c)
        pof.append(P)
    n = len(ctxs)
    tail = np.full((n, M), -1, dtype=np.int32)
    for b, c in enumerate(ctxs):
        c = c[-M:]
        tail[b, M - len(c):] = c
    slots = to_dev(np.arange(n, dtype=np.int32))
    ctx.bs_rollout_begin(slots, to_dev(np.arange(n, dtype=np.int64)), to_dev(np.asarray(pof, np.int32)),
                         to_dev(tail), to_dev(np.full(n, 1 << 20, dtype=np.int32)))
    d = torch.zeros((n, k), dtype=torch.int32, device="cuda")
    dl = torch.zeros(n, dtype=torch.int32, device="cuda")
    ml = torch.zeros(n, dtype=torch.int32, device="cuda")
    ctx.bs_draft_lookup(rl_step, slots, k, d, dl, ml)
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    d, dl, ml = d.cpu().numpy(), dl.cpu().numpy(), ml.cpu().numpy()
    for b in range(n):
        want, mstar = orc.lookup(pools.get(pof[b], []), ctxs[b][-M:], M, 1, k)
        assert int(dl[b]) == len(want), b
        assert [int(x) for x in d[b, : dl[b]]] == want, b
        assert int(ml[b]) == mstar, b


def test_exchange_one_rank_nccl(bs, orc):
    """A 1-rank NCCL communicator on one B200: the exchange keeps every sequence (owner(P) =
    P mod 1), runs the all-gathers and the device gather, and the sealed index answers
    lookups exactly like the oracle over the put pools."""
    vocab, k, M = 6, 8, 32
    sp, off, tok = _random_pools(11, 7, vocab)
    ctx = bs.Context(vocab=vocab, k_max=k, match_max=M, max_rollouts=128, pool_capacity_tokens=len(tok) + 8,
                     pool_capacity_seqs=len(sp) + 2)
    comm = bs.nccl_comm_init(bs.nccl_unique_id(), 1, 0)
    try:
        ctx.bs_draft_pool_put(3, to_dev(sp), to_dev(off), to_dev(tok), int(len(tok)))
        ctx.bs_draft_exchange(comm, 0, 1, 3)
        ctx.bs_draft_pool_seal(3)
        _lookup_vs_oracle(bs, orc, ctx, 3, (sp, off, tok), np.unique(sp), vocab, k, M, 5)
    finally:
        bs.nccl_comm_destroy(comm)


def _two_rank_worker(rank, world, uid, ret):
    import oracle as orc
    import paper_2605_08862_b200 as bs

    torch.cuda.set_device(rank)
    vocab, k, M = 5, 8, 32
    # rank r pre-generated drafts for prompts of both ranks (prompt ids r*100 + 0..5)
    sp, off, tok = _random_pools(21 + rank, 6, vocab, prompt_base=100 * rank)
    allp = [_random_pools(21 + r, 6, vocab, prompt_base=100 * r) for r in range(world)]
    ctx = bs.Context(vocab=vocab, k_max=k, match_max=M, max_rollouts=128, device=rank,
                     pool_capacity_tokens=sum(len(p[2]) for p in allp) + 8,
                     pool_capacity_seqs=sum(len(p[0]) for p in allp) + 2)
    comm = bs.nccl_comm_init(uid, world, rank)
    try:
        ctx.bs_draft_pool_put(4, to_dev(sp), to_dev(off), to_dev(tok), int(len(tok)))
        ctx.bs_draft_exchange(comm, rank, world, 4)
        ctx.bs_draft_pool_seal(4)
        # the pools this rank owns: every rank's sequences of prompts P with P % world == rank
        seqs, prm = [], []
        for p_sp, p_off, p_tok in allp:
            for i, P in enumerate(p_sp):
                if int(P) % world == rank:
                    seqs.append(p_tok[p_off[i]:p_off[i + 1]])
                    prm.append(int(P))
        o = np.zeros(len(seqs) + 1, dtype=np.int64)
        o[1:] = np.cumsum([len(s) for s in seqs])
        _lookup_vs_oracle(bs, orc, ctx, 4, (np.asarray(prm, np.int32), o, np.concatenate(seqs)),
                          np.unique(prm), vocab, k, M, 9 + rank)
        ret[rank] = "ok"
    finally:
        bs.nccl_comm_destroy(comm)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs 2 GPUs (NCCL refuses two ranks on one device)")
def test_exchange_two_ranks_nccl(bs):
    """World size 2 over NCCL (NVLink): each rank keeps the sequences of its own prompts from
    both ranks' pools; lookups equal the oracle over exactly those pools."""
    import torch.multiprocessing as tmp

    import paper_2605_08862_b200 as bsm

    uid = bsm.nccl_unique_id()
    ctx = tmp.get_context("spawn")
    mgr = ctx.Manager()
    ret = mgr.dict()
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    procs = [ctx.Process(target=_two_rank_worker, args=(r, 2, uid, ret)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert dict(ret) == {0: "ok", 1: "ok"}
