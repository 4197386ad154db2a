"""End-to-end parity of the decoding loop (lookup -> target rows -> verify -> commit):
RolloutEngine on the GPU vs the oracle's Alg. 1 loop, token for token."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import TargetSpec  # noqa: E402
from tests.gpu_util import bank_numpy, pools_for, setup_rollouts, to_dev  # noqa: E402
from paper_2605_08862_b200.engine import TARGET_MODES  # noqa: E402


def _engine(bs, spec, n, k, M, T, top_p, seed, eos, pool_tokens, pool_seqs, fused="lookup", top_k=0):
    from paper_2605_08862_b200.engine import RolloutEngine, Target

    ctx = bs.Context(vocab=spec.V, eos_id=eos, k_max=k, match_max=M, max_rollouts=n,
                     pool_capacity_tokens=max(1, pool_tokens), pool_capacity_seqs=max(1, pool_seqs),
                     seed=seed)
    bank = to_dev(bank_numpy(spec).view(np.int16))
    mode = TARGET_MODES[spec.mode]
    # "lookup": bs_verify_commit_lookup; "commit": lookup + bs_verify_commit; "none": lookup +
    # bs_verify_step + bs_commit
    eng = RolloutEngine(ctx, n, k, T, top_p, Target(bank, spec.nbank, spec.target_seed, mode),
                        fused=fused != "none", fuse_lookup=fused == "lookup", top_k=top_k)
    return ctx, eng


def _oracle_rollouts(orc, spec, pid, tail_rows, uids, ml, pools_np, k, M, T, top_p, seed, eos,
                     which, max_steps=None, top_k=0):
    from oracle.rollout import OracleRollout, bank_row_fn, pools_by_prompt, run_rollouts

    pools = pools_by_prompt(*pools_np)
    ros = [OracleRollout(prompt=int(pid[b]), uid=int(uids[b]),
                         context=[int(x) for x in tail_rows[b] if x >= 0], max_len=int(ml[b]))
           for b in which]
    run_rollouts(ros, pools, bank_row_fn(spec), k=k, M=M, Lmin=1, T=T, top_p=top_p, seed=seed,
                 eos=eos, max_steps=max_steps, top_k=top_k)
    return ros


@pytest.mark.parametrize("fused", ["lookup", "commit", "none"])
@pytest.mark.parametrize("T,mode", [(0.0, "markov"), (1.0, "markov"), (1.0, "mixed"),
                                    (0.7, "position")])
def test_tiny_rollouts_token_for_token(bs, orc, T, mode, fused):
    """TINY config: V=1024, 4 rollouts of one prompt, k=4, 64-token responses."""
    spec = TargetSpec(V=1024, nbank=256, mode=mode, beta=6.0)
    M, k, L, seed, eos = 16, 4, 64, 5, 1023
    prompts, tails, pid, tail_rows, uids, ml = setup_rollouts(spec, 1, 4, M, L)
    pools_np = pools_for(spec, prompts, tails, 4, np.full(4, 60), 0.85, prefix=M)
    n = len(pid)
    ctx, eng = _engine(bs, spec, n, k, M, T, 1.0, seed, eos, len(pools_np[2]), len(pools_np[0]),
                       fused=fused)
    resp = torch.full((n, L), -1, dtype=torch.int32, device="cuda")
    ctx.bs_rollout_bind_output(resp, L)
    eng.put_pools(1, to_dev(pools_np[0]), to_dev(pools_np[1]), to_dev(pools_np[2]))
    eng.seal(1)
    eng.begin(to_dev(uids.view(np.int64)), to_dev(pid), to_dev(tail_rows), to_dev(ml))
    steps = eng.run_until_done(chunk=8, use_graph=False)
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    got = resp.cpu().numpy()
    ros = _oracle_rollouts(orc, spec, pid, tail_rows, uids, ml, pools_np, k, M, T, 1.0, seed, eos,
                           range(n))
    n_spec = 0
    for b, ro in enumerate(ros):
        assert [int(x) for x in got[b, : len(ro.generated)]] == ro.generated, b
        assert all(x == -1 for x in got[b, len(ro.generated):])
        n_spec += sum(1 for s in ro.steps if s[0] > 0)
    st = eng.stats()
    assert st["verify_steps"] == n_spec
    assert st["tokens"] == sum(len(r.generated) for r in ros)
    assert n_spec > 0
    # every device counter behind AL / DL / AR equals the oracle's own
    # accounting of the same steps: (q, m*, draft, emitted, accepted, StepOut)
    steps_ = [s_ for ro in ros for s_ in ro.steps]
    vs = [s_ for s_ in steps_ if s_[0] > 0]
    assert st["plain_steps"] == len(steps_) - len(vs)
    assert st["accepted"] == sum(s_[4] for s_ in vs)
    assert st["proposed"] == sum(s_[0] for s_ in vs)
    assert st["rows_needed"] == sum(s_[5].rows_used for s_ in steps_)
    hist = [0] * len(st["streak_hist"])
    for s_ in vs:
        hist[min(len(s_[3]), len(hist) - 1)] += 1
    assert st["streak_hist"] == hist
    if st["verify_steps"]:
        assert st["acceptance_length"] == sum(len(s_[3]) for s_ in vs) / len(vs)


@pytest.mark.parametrize("top_k,top_p", [(5, 1.0), (40, 0.9)])
def test_tiny_rollouts_top_k(bs, orc, top_k, top_p):
    """TINY rollouts under top-k (then top-p) filtering (readings R5k, R5): the filtered verify
    kernel with its separate commit / lookup launches, token-for-token vs the oracle's loop."""
    spec = TargetSpec(V=1024, nbank=256, mode="mixed", beta=6.0)
    M, k, L, seed, eos = 16, 4, 48, 9, 1023
    prompts, tails, pid, tail_rows, uids, ml = setup_rollouts(spec, 1, 4, M, L)
    pools_np = pools_for(spec, prompts, tails, 4, np.full(4, 44), 0.85, prefix=M)
    n = len(pid)
    ctx, eng = _engine(bs, spec, n, k, M, 1.0, top_p, seed, eos, len(pools_np[2]), len(pools_np[0]),
                       top_k=top_k)
    resp = torch.full((n, L), -1, dtype=torch.int32, device="cuda")
    ctx.bs_rollout_bind_output(resp, L)
    eng.put_pools(1, to_dev(pools_np[0]), to_dev(pools_np[1]), to_dev(pools_np[2]))
    eng.seal(1)
    eng.begin(to_dev(uids.view(np.int64)), to_dev(pid), to_dev(tail_rows), to_dev(ml))
    eng.run_until_done(chunk=8, use_graph=True)
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    got = resp.cpu().numpy()
    ros = _oracle_rollouts(orc, spec, pid, tail_rows, uids, ml, pools_np, k, M, 1.0, top_p, seed, eos,
                           range(n), top_k=top_k)
    for b, ro in enumerate(ros):
        assert [int(x) for x in got[b, : len(ro.generated)]] == ro.generated, b
    assert eng.stats()["proposed"] > 0


@pytest.mark.parametrize("tau", [0.3, 0.6])
def test_tiny_rollouts_confidence_scored_drafts(bs, orc, tau):
    """TINY rollouts with confidence-scored suffix drafts (f4, reading C1: the index build stops
    each greedy descent at the first child below min_token_prob), fused verify + commit + lookup
    under graph replay: token-for-token vs the oracle's loop with the same threshold, and fewer
    drafted tokens than without the threshold."""
    spec = TargetSpec(V=1024, nbank=256, mode="position", beta=12.0)
    M, k, L, seed, eos = 16, 4, 48, 21, -1
    prompts, tails, pid, tail_rows, uids, ml = setup_rollouts(spec, 2, 3, M, L)
    pools_np = pools_for(spec, prompts, tails, 4, np.full(8, 44), 0.7, prefix=M)
    n = len(pid)
    ctx, eng = _engine(bs, spec, n, k, M, 1.0, 1.0, seed, eos, len(pools_np[2]), len(pools_np[0]))
    ctx.bs_draft_set_min_token_prob(tau)
    resp = torch.full((n, L), -1, dtype=torch.int32, device="cuda")
    ctx.bs_rollout_bind_output(resp, L)
    eng.put_pools(1, to_dev(pools_np[0]), to_dev(pools_np[1]), to_dev(pools_np[2]))
    eng.seal(1)
    eng.begin(to_dev(uids.view(np.int64)), to_dev(pid), to_dev(tail_rows), to_dev(ml))
    eng.run_until_done(chunk=8, use_graph=True)
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    got = resp.cpu().numpy()
    from oracle.rollout import OracleRollout, bank_row_fn, pools_by_prompt, run_rollouts

    def oracle_run(t):
        ros = [OracleRollout(prompt=int(pid[b]), uid=int(uids[b]),
                             context=[int(x) for x in tail_rows[b] if x >= 0], max_len=int(ml[b]))
               for b in range(n)]
        run_rollouts(ros, pools_by_prompt(*pools_np), bank_row_fn(spec), k=k, M=M, Lmin=1, T=1.0,
                     top_p=1.0, seed=seed, eos=eos, min_token_prob=t)
        return ros

    ros = oracle_run(tau)
    for b, ro in enumerate(ros):
        assert [int(x) for x in got[b, : len(ro.generated)]] == ro.generated, b
    st = eng.stats()
    assert st["accepted"] == sum(s_[4] for ro in ros for s_ in ro.steps)
    assert st["proposed"] == sum(s_[0] for ro in ros for s_ in ro.steps)
    plain = oracle_run(0.0)
    assert st["proposed"] / st["decode_steps"] < (sum(s_[0] for ro in plain for s_ in ro.steps)
                                                  / sum(len(ro.steps) for ro in plain))


@pytest.mark.parametrize("ngram", [(1, 4), (2, 8)])
def test_tiny_rollouts_ngram_drafts(bs, orc, ngram):
    """TINY rollouts drafted by the n-gram linear-scan drafter (f4, reading N1) under graph
    replay: token-for-token vs the oracle's loop with the same drafter; drafts accepted."""
    spec = TargetSpec(V=1024, nbank=256, mode="position", beta=12.0)
    M, k, L, seed, eos = 16, 4, 48, 21, -1
    prompts, tails, pid, tail_rows, uids, ml = setup_rollouts(spec, 2, 3, M, L)
    pools_np = pools_for(spec, prompts, tails, 4, np.full(8, 44), 0.85, prefix=M)
    n = len(pid)
    ctx, eng = _engine(bs, spec, n, k, M, 1.0, 1.0, seed, eos, len(pools_np[2]), len(pools_np[0]))
    eng.ngram = ngram
    eng.fuse_lookup = False
    resp = torch.full((n, L), -1, dtype=torch.int32, device="cuda")
    ctx.bs_rollout_bind_output(resp, L)
    eng.put_pools(1, to_dev(pools_np[0]), to_dev(pools_np[1]), to_dev(pools_np[2]))
    eng.seal(1)
    eng.begin(to_dev(uids.view(np.int64)), to_dev(pid), to_dev(tail_rows), to_dev(ml))
    eng.run_until_done(chunk=8, use_graph=True)
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    got = resp.cpu().numpy()
    from oracle.rollout import OracleRollout, bank_row_fn, pools_by_prompt, run_rollouts

    ros = [OracleRollout(prompt=int(pid[b]), uid=int(uids[b]), context=[int(x) for x in tail_rows[b] if x >= 0],
                         max_len=int(ml[b])) for b in range(n)]
    run_rollouts(ros, pools_by_prompt(*pools_np), bank_row_fn(spec), k=k, M=M, Lmin=1, T=1.0, top_p=1.0,
                 seed=seed, eos=eos, ngram=ngram)
    for b, ro in enumerate(ros):
        assert [int(x) for x in got[b, : len(ro.generated)]] == ro.generated, b
    st = eng.stats()
    assert st["accepted"] > 0
    assert st["accepted"] == sum(s_[4] for ro in ros for s_ in ro.steps)


def test_tiny_rollouts_graph_replay_matches_eager(bs, orc):
    """The CUDA-graph multi-step loop emits exactly what eager stepping emits."""
    spec = TargetSpec(V=1024, nbank=256, mode="mixed", beta=6.0)
    M, k, L, seed = 16, 4, 64, 9
    prompts, tails, pid, tail_rows, uids, ml = setup_rollouts(spec, 2, 4, M, L)
    pools_np = pools_for(spec, prompts, tails, 4, np.full(8, 60), 0.85, prefix=M)
    outs = []
    for use_graph in (False, True):
        n = len(pid)
        ctx, eng = _engine(bs, spec, n, k, M, 1.0, 1.0, seed, -1, len(pools_np[2]), len(pools_np[0]))
        resp = torch.full((n, L), -1, dtype=torch.int32, device="cuda")
        ctx.bs_rollout_bind_output(resp, L)
        eng.put_pools(1, to_dev(pools_np[0]), to_dev(pools_np[1]), to_dev(pools_np[2]))
        eng.seal(1)
        eng.begin(to_dev(uids.view(np.int64)), to_dev(pid), to_dev(tail_rows), to_dev(ml))
        eng.run_until_done(chunk=8, use_graph=use_graph)
        torch.cuda.synchronize()
        outs.append(resp.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


def test_qwen_shaped_sampled_parity(bs, orc):
    """Q7 config at full size (V=151936, 256 rollouts, k=8, the bench's launch path):
    sampled rollouts checked against the oracle for their first 3 decoding steps."""
    spec = TargetSpec(V=151936, nbank=512, mode="position", beta=12.0)
    M, k, seed = 32, 8, 17
    prompts, tails, pid, tail_rows, uids, ml = setup_rollouts(spec, 16, 16, M, 4096)
    rng = np.random.default_rng(0)
    pools_np = pools_for(spec, prompts, tails, 16, rng.integers(100, 600, 256), 0.9, prefix=M)
    n = len(pid)
    ctx, eng = _engine(bs, spec, n, k, M, 1.0, 1.0, seed, -1, len(pools_np[2]), len(pools_np[0]))
    resp = torch.full((n, 64), -1, dtype=torch.int32, device="cuda")
    ctx.bs_rollout_bind_output(resp, 64)
    eng.put_pools(1, to_dev(pools_np[0]), to_dev(pools_np[1]), to_dev(pools_np[2]))
    eng.seal(1)
    eng.begin(to_dev(uids.view(np.int64)), to_dev(pid), to_dev(tail_rows), to_dev(ml))
    for _ in range(3):
        eng.step()
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    got = resp.cpu().numpy()
    which = [0, 37, 128, 201, 255]
    ros = _oracle_rollouts(orc, spec, pid, tail_rows, uids, ml, pools_np, k, M, 1.0, 1.0, seed, -1,
                           which, max_steps=3)
    for b, ro in zip(which, ros):
        assert [int(x) for x in got[b, : len(ro.generated)]] == ro.generated, b
    st = eng.stats()
    assert st["verify_steps"] > 0 and st["accepted"] > 0


def _run_engine(bs, spec, pid, tail_rows, uids, ml, pools_np, k, M, T, top_p, seed, fused, steps, chunk):
    n = len(pid)
    ctx, eng = _engine(bs, spec, n, k, M, T, top_p, seed, -1, len(pools_np[2]), len(pools_np[0]),
                       fused=fused)
    L = int(ml.max())
    resp = torch.full((n, L), -1, dtype=torch.int32, device="cuda")
    ctx.bs_rollout_bind_output(resp, L)
    eng.put_pools(1, to_dev(pools_np[0]), to_dev(pools_np[1]), to_dev(pools_np[2]))
    eng.seal(1)
    eng.begin(to_dev(uids.view(np.int64)), to_dev(pid), to_dev(tail_rows), to_dev(ml))
    if chunk:
        eng.capture(chunk)  # (runs one eager step first)
        for _ in range(steps // chunk):
            eng.run_graph()
    else:
        for _ in range(steps):
            eng.step()
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    if fused != "lookup":  # the next step's drafts, as the fused launch leaves them
        ctx.bs_draft_lookup(eng.rl_step, eng.slots, k, eng.draft, eng.draft_len, eng.match_len,
                            stream=eng.stream)
        torch.cuda.synchronize()
    st = eng.stats()
    return dict(resp=resp.cpu().numpy(), draft=eng.draft.cpu().numpy(), dlen=eng.draft_len.cpu().numpy(),
                mlen=eng.match_len.cpu().numpy(), fin=eng.finished.cpu().numpy(), st=st)


@pytest.mark.parametrize("top_p", [1.0, 0.9])  # 0.9: the unfused fallback (verify, commit, lookup kernels)
def test_fused_lookup_matches_separate_lookup_tiny(bs, top_p):
    """bs_verify_commit_lookup leaves exactly the state, responses and next drafts of
    bs_verify_commit + bs_draft_lookup (short rollouts: most finish inside the run)."""
    spec = TargetSpec(V=1024, nbank=256, mode="position", beta=12.0)  # p_peak ~0.9: long accepts
    M, k, seed = 16, 4, 21
    ml_ = np.random.default_rng(3).integers(8, 60, 16)
    prompts, tails, pid, tail_rows, uids, ml = setup_rollouts(spec, 2, 8, M, ml_)
    pools_np = pools_for(spec, prompts, tails, 8, np.full(16, 60), 0.85, prefix=M)
    a = _run_engine(bs, spec, pid, tail_rows, uids, ml, pools_np, k, M, 1.0, top_p, seed, "commit", 40, 0)
    b = _run_engine(bs, spec, pid, tail_rows, uids, ml, pools_np, k, M, 1.0, top_p, seed, "lookup", 40, 0)
    for key in ("resp", "draft", "dlen", "mlen", "fin"):
        assert np.array_equal(a[key], b[key]), key
    drop = lambda d: {x: v for x, v in d.items() if x != "rows_verified"}  # noqa: E731 (speculation)
    assert drop(a["st"]) == drop(b["st"])
    assert a["fin"].sum() > 0 and a["st"]["accepted"] > 0


def test_fused_lookup_matches_separate_lookup_q7(bs):
    """Q7 shape (V=151936, 256 rollouts, k=8), the bench's launch path (CUDA graph chunks):
    fused and separate lookups give identical responses, drafts and statistics."""
    spec = TargetSpec(V=151936, nbank=512, mode="position", beta=12.0)
    M, k, seed = 32, 8, 23
    prompts, tails, pid, tail_rows, uids, ml = setup_rollouts(spec, 16, 16, M, 160)
    rng = np.random.default_rng(1)
    pools_np = pools_for(spec, prompts, tails, 16, rng.integers(60, 200, 256), 0.9, prefix=M)
    a = _run_engine(bs, spec, pid, tail_rows, uids, ml, pools_np, k, M, 1.0, 1.0, seed, "commit", 64, 16)
    b = _run_engine(bs, spec, pid, tail_rows, uids, ml, pools_np, k, M, 1.0, 1.0, seed, "lookup", 64, 16)
    for key in ("resp", "draft", "dlen", "mlen", "fin"):
        assert np.array_equal(a[key], b[key]), key
    drop = lambda d: {x: v for x, v in d.items() if x != "rows_verified"}  # noqa: E731 (speculation)
    assert drop(a["st"]) == drop(b["st"])
    assert a["st"]["accepted"] > 0 and (a["mlen"] > 0).any()


@pytest.mark.parametrize("fused", ["lookup", "none"])
def test_graph_replay_staleness_on_device(bs, fused):
    """SPEC S:340 (a lookup against a pool sealed for another RL step is a hard error) under
    CUDA-graph replay, where the host-side rl_step check cannot run: a put for a new step
    without its seal makes every replayed lookup stale on the device (empty drafts,
    BS_DEV_STALE -> BS_ERR_STALE); after the seal the same graph replays cleanly; a repeated
    seal of the sealed step is a no-op."""
    spec = TargetSpec(V=1024, nbank=64, mode="mixed", beta=6.0)
    M, k, L = 16, 4, 4000
    prompts, tails, pid, tail_rows, uids, ml = setup_rollouts(spec, 2, 4, M, L)
    pools_np = pools_for(spec, prompts, tails, 4, np.full(8, 300), 0.9, prefix=M)
    n = len(pid)
    ctx, eng = _engine(bs, spec, n, k, M, 1.0, 1.0, 7, -1, 2 * len(pools_np[2]), 2 * len(pools_np[0]),
                       fused=fused)
    put = lambda s: eng.put_pools(s, to_dev(pools_np[0]), to_dev(pools_np[1]), to_dev(pools_np[2]))  # noqa: E731
    put(1)
    eng.seal(1)
    eng.begin(to_dev(uids.view(np.int64)), to_dev(pid), to_dev(tail_rows), to_dev(ml))
    eng.capture(4)
    eng.run_graph()
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    assert eng.stats(reset=True)["proposed"] > 0  # the sealed index serves drafts
    put(2)  # a new RL step's pools: the step-1 index is stale until the step-2 seal
    eng.run_graph()
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() & 0x20  # BS_DEV_STALE
    st = eng.stats(reset=True)
    # empty drafts: plain decoding only (fused lookup: the replay's first step still uses the
    # drafts looked up before the put)
    assert st["proposed"] <= (n * k if fused == "lookup" else 0) and st["tokens"] > 0
    eng.seal(2)
    eng.seal(2)  # repeated seal of the sealed step: a no-op, the index keeps its pools
    eng.run_graph()
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    assert eng.stats(reset=True)["proposed"] > 0
