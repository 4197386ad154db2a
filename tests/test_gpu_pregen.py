"""f1: bubble pre-generation with the polling synchronizer.

- the synchronizer's arrive / poll semantics (halt once ALL ranks completed B_t);
- pre-generation is plain decoding (Alg. 1 lines 4-7) of the next step's prompts: its tokens
  equal the oracle's plain decoding with the same uids (empty pool), chunk by chunk;
- a poll inside the chunk graph halts pre-generation after the last rank arrives;
- the pre-generated responses, as pools, feed the next RL step: its drafts are accepted and its
  rollouts match the oracle run on the same pools;
- across two processes on two GPUs (CUDA IPC over NVLink) when two GPUs exist.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from workloads import TargetSpec  # noqa: E402

from tests.gpu_util import bank_numpy, setup_rollouts, to_dev  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bubble_sync_arrive_poll(bs):
    s = bs.BubbleSync(0)
    halt = torch.full((1,), -1, dtype=torch.int32, device="cuda")

    def poll(world, step):
        s.poll(world, step, halt)
        torch.cuda.synchronize()
        return int(halt.item())

    assert poll(1, 0) == 0                   # nobody finished anything yet
    s.arrive(0, 7)
    assert poll(1, 7) == 1 and poll(1, 5) == 1 and poll(1, 8) == 0
    assert poll(2, 7) == 0                   # rank 1 still decoding B_7
    s.arrive(1, 7)
    assert poll(2, 7) == 1 and poll(3, 7) == 0
    s.arrive(0, 8)
    assert poll(2, 8) == 0                   # words are monotone: no reset between RL steps
    s.arrive(1, 8)
    assert poll(2, 8) == 1
    with pytest.raises(bs.BubbleSpecError):
        s.arrive(64, 1)
    s.close()


def _setup(bs, spec, n_main, n_pre, M, L, seed):
    from paper_2605_08862_b200.engine import TARGET_MODES, Target

    ctx = bs.Context(vocab=spec.V, eos_id=-1, k_max=4, match_max=M, max_rollouts=n_main + n_pre,
                     pool_capacity_tokens=1 << 16, pool_capacity_seqs=256, seed=seed)
    bank = to_dev(bank_numpy(spec).view(np.int16))
    target = Target(bank, spec.nbank, spec.target_seed, TARGET_MODES[spec.mode])
    resp = torch.full((n_main + n_pre, L), -1, dtype=torch.int32, device="cuda")
    ctx.bs_rollout_bind_output(resp, L)
    return ctx, target, resp


def _oracle_plain(spec, pid, tails, uids, ml, seed, steps=None, pools=None, k=0, M=16):
    from oracle.rollout import OracleRollout, bank_row_fn, run_rollouts

    ros = [OracleRollout(prompt=int(pid[b]), uid=int(uids[b]), context=[int(x) for x in tails[b] if x >= 0],
                         max_len=int(ml[b])) for b in range(len(pid))]
    run_rollouts(ros, pools or {}, bank_row_fn(spec), k=k, M=M, Lmin=1, T=1.0, top_p=1.0, seed=seed, eos=-1,
                 max_steps=steps)
    return ros


def test_pregen_is_plain_decoding_and_halts(bs, orc):
    spec = TargetSpec(V=1024, nbank=256, mode="position", beta=10.0)
    M, L, seed, n_pre = 16, 400, 13, 6
    ctx, target, resp = _setup(bs, spec, 4, n_pre, M, L, seed)
    sync = bs.BubbleSync(0)
    pre = bs.Pregenerator(ctx, 4, n_pre, target, sync, rank=0, world=2, poll_every=5)
    _, _, pid, tails, uids, ml = setup_rollouts(spec, 2, 3, M, L, seed=4)
    pre.begin(to_dev(uids.view(np.int64)), to_dev(pid), to_dev(tails), to_dev(ml))
    sync.arrive(0, 3)  # this rank finished B_3; rank 1 has not: pre-generation runs
    steps = pre.run(3, max_chunks=4)
    assert steps == 1 + 4 * 5  # the capture's warm step, then 4 chunks of T = 5
    sync.arrive(1, 3)  # the last rank finishes B_3: the next chunk's poll halts
    steps2 = pre.run(3)
    assert steps2 == steps + 5
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    got = resp.cpu().numpy()[4:]
    ros = _oracle_plain(spec, pid, tails, uids, ml, seed, steps=steps2)
    for b, ro in enumerate(ros):
        assert len(ro.generated) == steps2
        assert [int(x) for x in got[b, :steps2]] == ro.generated, b
        assert all(x == -1 for x in got[b, steps2:])
    sp, off, tok = pre.pools(pid, tails, got, M)
    assert len(sp) == n_pre and int(off[-1]) == n_pre * (M + steps2)
    sync.close()


def test_pregen_pools_feed_next_step(bs, orc):
    """The BubbleSpec loop on one GPU: B_t's rank pre-generates the next prompts until the
    synchronizer halts it, the responses become B_{t+1}'s pools, and B_{t+1}'s speculative
    rollouts (fused verify + commit + lookup) accept drafts and equal the oracle's on the same
    pools."""
    from oracle.rollout import pools_by_prompt
    from paper_2605_08862_b200.engine import RolloutEngine

    spec = TargetSpec(V=1024, nbank=256, mode="position", beta=12.0)
    M, L, seed, k = 16, 96, 17, 4
    _, _, pid, tails, uids, ml = setup_rollouts(spec, 2, 4, M, L, seed=9)
    n = len(pid)
    ctx, target, resp = _setup(bs, spec, n, n, M, L, seed)
    sync = bs.BubbleSync(0)
    pre = bs.Pregenerator(ctx, n, n, target, sync, rank=0, world=2, poll_every=8)
    pre_uids = uids + np.uint64(1 << 40)  # the pre-generation samples are other rollouts
    pre.begin(to_dev(pre_uids.view(np.int64)), to_dev(pid), to_dev(tails), to_dev(ml))
    sync.arrive(0, 0)
    pre.run(0, max_chunks=6)
    sync.arrive(1, 0)
    pre.run(0)
    torch.cuda.synchronize()
    got_pre = resp.cpu().numpy()[n:]
    sp, off, tok = pre.pools(pid, tails, got_pre, M)
    assert len(sp) == n
    # next RL step: its rollouts (new uids) draft from the pre-generated pools
    eng = RolloutEngine(ctx, n, k, 1.0, 1.0, target)
    eng.put_pools(1, to_dev(sp), to_dev(off), to_dev(tok))
    eng.seal(1)
    eng.begin(to_dev(uids.view(np.int64)), to_dev(pid), to_dev(tails), to_dev(ml))
    eng.run_until_done(chunk=8)
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    st = eng.stats()
    assert st["accepted"] > 0 and st["acceptance_length"] > 1.2
    got = resp.cpu().numpy()[:n]
    ros = _oracle_plain(spec, pid, tails, uids, ml, seed, pools=pools_by_prompt(sp, off, tok), k=k, M=M)
    for b, ro in enumerate(ros):
        assert [int(x) for x in got[b, : len(ro.generated)]] == ro.generated, b
    sync.close()


def test_pregen_two_processes_ipc(bs):
    """Rank 1 (its own process and GPU) arrives on rank 0's synchronizer over NVLink; rank 0's
    poll sees it."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29611")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29611",
                        os.path.join(ROOT, "tests", "pregen_ipc_worker.py")],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "ipc poll ok" in r.stdout
