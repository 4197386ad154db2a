"""End-to-end parity of the decoding loop (lookup -> target rows -> verify -> commit):
RolloutEngine on the GPU vs the oracle's Alg. 1 loop, token for token."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import TargetSpec  # noqa: E402
from tests.gpu_util import bank_numpy, pools_for, setup_rollouts, to_dev  # noqa: E402


def _engine(bs, spec, n, k, M, T, top_p, seed, eos, pool_tokens, pool_seqs, fused=True):
    from paper_2605_08862_b200.engine import RolloutEngine, Target

    ctx = bs.Context(vocab=spec.V, eos_id=eos, k_max=k, match_max=M, max_rollouts=n,
                     pool_capacity_tokens=max(1, pool_tokens), pool_capacity_seqs=max(1, pool_seqs),
                     seed=seed)
    bank = to_dev(bank_numpy(spec).view(np.int16))
    mode = {"position": 0, "markov": 1, "mixed": 2}[spec.mode]
    eng = RolloutEngine(ctx, n, k, T, top_p, Target(bank, spec.nbank, spec.target_seed, mode),
                        fused=fused)
    return ctx, eng


def _oracle_rollouts(orc, spec, pid, tail_rows, uids, ml, pools_np, k, M, T, top_p, seed, eos,
                     which, max_steps=None):
    from oracle.rollout import OracleRollout, bank_row_fn, pools_by_prompt, run_rollouts

    pools = pools_by_prompt(*pools_np)
    ros = [OracleRollout(prompt=int(pid[b]), uid=int(uids[b]),
                         context=[int(x) for x in tail_rows[b] if x >= 0], max_len=int(ml[b]))
           for b in which]
    run_rollouts(ros, pools, bank_row_fn(spec), k=k, M=M, Lmin=1, T=T, top_p=top_p, seed=seed,
                 eos=eos, max_steps=max_steps)
    return ros


@pytest.mark.parametrize("fused", [True, False])  # bs_verify_commit vs bs_verify_step + bs_commit
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
