"""N > 1 path on CPU: the cross-rank draft exchange with world
size 2 over gloo.  Each rank produces pools for the OTHER rank's prompts (drafts made in its
bubble), the padded metadata/payload is all-gathered exactly as bs_draft_exchange does over
NCCL, and the library's host routing plan (bs_route_plan) decides what each rank keeps.
Checked: every rank keeps exactly the sequences of the prompts it owns (prompt % world ==
rank), byte-identical, and the union over ranks is everything that was produced."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_pools(rank, world, source="perturbed"):
    from workloads import TargetSpec, make_pools, prompt_tails

    spec = TargetSpec(V=1000, nbank=64)
    prod_for = (rank + 1) % world
    prompts = np.array([i * world + prod_for for i in range(3)], dtype=np.int64)
    tails = prompt_tails(5, prompts, 8, spec.V)
    lens = np.random.default_rng(rank).integers(0, 30, (3, 4))
    if source == "pregen":
        # f1: the responses this rank pre-generated in its bubble for the next prompts (4 per
        # prompt, some empty: the synchronizer halted them early), as pool sequences
        from paper_2605_08862_b200.pregen import pool_sequences

        pid = np.repeat(prompts, 4).astype(np.int32)
        trows = np.repeat(tails, 4, axis=0)
        resp = np.random.default_rng(100 + rank).integers(0, spec.V, (12, 30)).astype(np.int32)
        return pool_sequences(pid, trows, resp, lens.ravel(), M=8)
    return make_pools(spec, prompts, tails, 4, lens, 0.8, prefix=8)


def _worker(rank, world, port, q, source="perturbed"):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_08862_b200 import bs_route_plan

        sp, off, tok = _rank_pools(rank, world, source)
        cnt = torch.tensor([len(sp), len(tok)], dtype=torch.int64)
        allc = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allc, cnt)
        counts = torch.stack(allc).numpy().ravel()
        max_seqs, max_tok = int(counts[0::2].max()), int(counts[1::2].max())
        o = torch.zeros(max_seqs + 1, dtype=torch.int64)
        o[: len(off)] = torch.from_numpy(off)
        p = torch.zeros(max(max_seqs, 1), dtype=torch.int32)
        p[: len(sp)] = torch.from_numpy(sp)
        t = torch.zeros(max(max_tok, 1), dtype=torch.int32)
        t[: len(tok)] = torch.from_numpy(tok)
        go = [torch.zeros_like(o) for _ in range(world)]
        gp = [torch.zeros_like(p) for _ in range(world)]
        gt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(go, o)
        dist.all_gather(gp, p)
        dist.all_gather(gt, t)
        offs = torch.stack(go).numpy().ravel()
        prm = torch.stack(gp).numpy().ravel()
        toks = torch.stack(gt).numpy().ravel()
        src, dst, ln, pr, ntok = bs_route_plan(world, rank, counts, offs, prm, max_seqs,
                                               max(max_tok, 1))
        kept = [(int(P), toks[s:s + n].tolist()) for s, n, P in zip(src, ln, pr)]
        q.put((rank, kept, int(ntok), [int(x) for x in dst]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("source", ["perturbed", "pregen"])
def test_exchange_routing_world2(source):
    """source "pregen": the pools are f1's pre-generated responses (pregen.pool_sequences)."""
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, source)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, kept, ntok, dst = q.get(timeout=120)
        res[r] = (kept, ntok, dst)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    produced = []
    for r in range(world):
        sp, off, tok = _rank_pools(r, world, source)
        produced += [(int(P), tok[off[s]:off[s + 1]].tolist()) for s, P in enumerate(sp)]
    union = []
    for r in range(world):
        kept, ntok, dst = res[r]
        assert all(P % world == r for P, _ in kept)
        assert ntok == sum(len(s) for _, s in kept)
        assert dst == list(np.cumsum([len(s) for _, s in kept]) - [len(s) for _, s in kept])
        union += kept
    assert sorted(union) == sorted(produced)
    # every rank owns something: pools produced by rank r are for rank r+1's prompts
    assert all(len(res[r][0]) > 0 for r in range(world))
