"""f1 measurement on one GPU: R virtual DP ranks (one context + stream + verify grid of
clusters/R each, decoding concurrently), the BubbleSpec loop of P:165-185 end to end:

  RL step t, every rank: put the pools pre-generated for its prompts during step t-1 (rank r
  pre-generates for rank (r+1) % R's next prompts: the exchange's routing, done here by
  putting into the owner's context), seal, decode its batch B_t (speculative, fused verify +
  commit + lookup graphs); when its batch is done it arrives on the synchronizer and
  pre-generates B_{t+1}'s prompts in chunks of T = 50 plain steps, each chunk ending with a
  poll, until every rank has arrived.

Step 0 has no pools (plain decoding: every step is one sample); later steps draft from the
previous step's bubbles.  Prints, per RL step: wall time (CUDA events), decode steps of the
slowest rank (the step count that sets rollout time), AL, pre-generated tokens, and the
bubble fraction (time ranks spent pre-generating / (R x step time)).

  python scripts/bubble_pregen.py [--ranks 4] [--steps 3] [--mean-len 2048]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_08862_b200 as bs  # noqa: E402
from paper_2605_08862_b200.engine import TARGET_MODES, RolloutEngine, Target  # noqa: E402
from workloads import TargetSpec, lognormal_lengths, prompt_tails  # noqa: E402


def main(argv=None, quiet=False):
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=4)
    ap.add_argument("--prompts", type=int, default=4, help="prompts per rank")
    ap.add_argument("--G", type=int, default=16, help="rollouts per prompt (= pre-generation batch, P:183)")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--mean-len", type=int, default=2048)
    ap.add_argument("--V", type=int, default=151936)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--poll", type=int, default=50)
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--beta", type=float, default=15.75)
    a = ap.parse_args(argv)
    R, P, G, V, k, M = a.ranks, a.prompts, a.G, a.V, a.k, 32
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    spec = TargetSpec(V=V, nbank=131072, mode="sample", beta=a.beta)
    bank = torch.empty((spec.nbank, V), dtype=torch.int16, device=dev)
    bs.bsx_synth_bank(bank, spec.nbank, V, spec.bank_seed, spec.beta)
    target = Target(bank, spec.nbank, spec.target_seed, TARGET_MODES[spec.mode])
    n = P * G
    cap = 32768
    ctxs, mains, pres, resp = [], [], [], []
    sync = bs.BubbleSync(0)
    for r in range(R):
        ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=M, max_rollouts=2 * n,
                         pool_capacity_tokens=n * cap + 1024, pool_capacity_seqs=n + 16, device=0, seed=0x5EED)
        ctx.bsx_set_max_clusters(max(1, 33 // R))
        st = torch.cuda.Stream(dev)
        rb = torch.full((2 * n, cap), -1, dtype=torch.int32, device=dev)
        ctx.bs_rollout_bind_output(rb, cap)
        ctxs.append(ctx)
        resp.append(rb)
        mains.append(RolloutEngine(ctx, n, k, 1.0, 1.0, target, stream=st))
        pres.append(bs.Pregenerator(ctx, n, n, target, sync, rank=r, world=R, poll_every=a.poll, stream=st))

    def batch(step, r):
        """Prompts of rank r at RL step `step` and their rollouts' metadata (host)."""
        prompts = np.array([step * 100_000 + i * R + r for i in range(P)], dtype=np.int64)
        tails = prompt_tails(7, prompts, M, V)
        pid = np.repeat(prompts, G).astype(np.int32)
        trows = np.repeat(tails, G, axis=0).astype(np.int32)
        ml = lognormal_lengths(1000 * step + r, n, a.mean_len, 0.6, cap).astype(np.int32)
        return pid, trows, ml

    def dev_t(x):
        return torch.from_numpy(np.ascontiguousarray(x)).to(dev)

    pools = [None] * R  # pools for rank r's prompts of the coming step
    flags = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in range(R)]
    report = []
    for step in range(a.steps):
        for r in range(R):
            ctx, eng = ctxs[r], mains[r]
            if pools[r] is None or len(pools[r][0]) == 0:  # no pools: a 1-token sequence of an unused prompt
                sp, off, tok = np.array([1 << 30], np.int32), np.array([0, 1], np.int64), np.array([0], np.int32)
            else:
                sp, off, tok = pools[r]
            eng.put_pools(step + 1, dev_t(sp), dev_t(off), dev_t(tok))
            eng.seal(step + 1)
            pid, trows, ml = batch(step, r)
            uids = (np.uint64(step) << np.uint64(32)) + np.uint64(r << 20) + np.arange(n, dtype=np.uint64)
            eng.begin(dev_t(uids.view(np.int64)), dev_t(pid), dev_t(trows), dev_t(ml))
            ctx.bs_stats_read(reset=True, stream=eng.stream)
            if eng.graph is None:
                eng.capture(a.chunk)
        torch.cuda.synchronize()
        t0 = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        t_done = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        t_halt = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        for r in range(R):
            t0[r].record(mains[r].stream)
        state = ["main"] * R
        main_steps = [0] * R
        next_b = [batch(step + 1, (r + 1) % R) for r in range(R)]
        wall0 = time.time()
        while any(s != "halt" for s in state):
            for r in range(R):
                eng, pre = mains[r], pres[r]
                if state[r] == "main":
                    with torch.cuda.stream(eng.stream):
                        eng.graph.replay()
                        main_steps[r] += a.chunk
                        flags[r].copy_(eng.live_count(), non_blocking=True)  # live rollouts
                elif state[r] == "pregen":
                    with torch.cuda.stream(pre.stream):
                        pre.graph.replay()
                        pre.steps += a.poll
                        flags[r].copy_(pre.halt, non_blocking=True)
            for r in range(R):
                if state[r] == "halt":
                    continue
                s = mains[r].stream
                s.synchronize()
                if state[r] == "main" and int(flags[r][0]) == 0:  # the batch is done
                    t_done[r].record(s)
                    sync.arrive(r, step, stream=s)
                    pid, trows, ml = next_b[r]
                    uids = (np.uint64(step + 1) << np.uint64(32)) + np.uint64(1 << 30) + np.uint64(r << 20) \
                        + np.arange(n, dtype=np.uint64)
                    pres[r].begin(dev_t(uids.view(np.int64)), dev_t(pid), dev_t(trows), dev_t(ml))
                    pres[r].run(step, max_chunks=0)  # capture (one warm step + a poll) only
                    state[r] = "pregen"
                    with torch.cuda.stream(s):
                        flags[r].copy_(pres[r].halt, non_blocking=True)
                    s.synchronize()
                    if int(flags[r][0]):
                        state[r] = "halt"
                        t_halt[r].record(s)
                elif state[r] == "pregen" and int(flags[r][0]):
                    state[r] = "halt"
                    t_halt[r].record(s)
        torch.cuda.synchronize()
        wall = time.time() - wall0
        step_ms = max(t0[r].elapsed_time(t_halt[r]) for r in range(R))
        done_ms = [t0[r].elapsed_time(t_done[r]) for r in range(R)]
        bubble_ms = [t_done[r].elapsed_time(t_halt[r]) for r in range(R)]
        stats = [mains[r].stats(reset=True) for r in range(R)]
        pre_tokens = 0
        for r in range(R):
            pid, trows, ml = next_b[r]
            got = resp[r][n:].cpu().numpy()
            sp, off, tok = pres[r].pools(pid, trows, got, M)
            pre_tokens += int(off[-1]) - M * len(sp)
            pools[(r + 1) % R] = (sp, off, tok)  # routed to the owner of those prompts
        tokens = sum(s_["tokens"] for s_ in stats)
        vsteps = sum(s_["verify_steps"] for s_ in stats)
        rec = {"rl_step": step, "step_ms": step_ms, "wall_s": wall, "rank_done_ms": done_ms,
               "bubble_ms": bubble_ms, "bubble_frac": sum(bubble_ms) / (R * step_ms),
               "slowest_rank_decode_steps": max(main_steps),  # graph-chunk granular (64)
               "mean_decode_steps_per_rollout": sum(s_["decode_steps"] for s_ in stats) / (R * n),
               "tokens": tokens,
               "acceptance_length": (sum((s_["acceptance_length"] or 0) * s_["verify_steps"] for s_ in stats)
                                     / vsteps) if vsteps else None,
               "verify_steps": vsteps, "plain_steps": sum(s_["plain_steps"] for s_ in stats),
               "pregen_tokens": pre_tokens, "tokens_per_s": tokens / (step_ms / 1e3)}
        report.append(rec)
        if not quiet:
            print(json.dumps(rec), flush=True)
        for r in range(R):
            assert ctxs[r].bs_sync_status() == 0
    first, last = report[0], report[-1]
    summary = {"summary": True, "ranks": R, "rollouts_per_rank": n, "mean_len": a.mean_len,
                      "decode_step_reduction_slowest_rank": 1 - last["slowest_rank_decode_steps"]
                      / first["slowest_rank_decode_steps"],
                      "decode_step_reduction_per_rollout": 1 - last["mean_decode_steps_per_rollout"]
                      / first["mean_decode_steps_per_rollout"],
                      "speedup_step_time": first["step_ms"] / last["step_ms"],
                      "bubble_frac_step0": first["bubble_frac"]}
    if not quiet:
        print(json.dumps(summary), flush=True)
    sync.close()
    return summary, report


if __name__ == "__main__":
    main()
