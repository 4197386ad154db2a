"""Fixed per-iteration cost of each decode op inside a CUDA graph, with every rollout
finished (zero live work) and with a handful live: 64 iterations of one op per graph,
timed as a whole (no event nodes inside), against a graph of trivial torch kernels."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2605_08862_b200 as bs  # noqa: E402
from paper_2605_08862_b200.engine import RolloutEngine, Target  # noqa: E402

cfg = bench.CONFIGS["q7"]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
stream = torch.cuda.Stream(dev)
V, k = cfg["V"], cfg["k"]
n = cfg["prompts"] * cfg["G"]
h = bench.make_step_inputs(cfg, 0, 0, 1)
ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=cfg["M"], max_rollouts=n,
                 pool_capacity_tokens=len(h["tokens"]) + 16,
                 pool_capacity_seqs=len(h["seq_prompt"]) + 4, seed=0x5EED)
spec = h["spec"]
bank = torch.empty((cfg["nbank"], V), dtype=torch.int16, device=dev)
bs.bsx_synth_bank(bank, cfg["nbank"], V, spec.bank_seed, spec.beta, stream=stream)
eng = RolloutEngine(ctx, n, k, cfg["T"], cfg["top_p"], Target(bank, cfg["nbank"], spec.target_seed, 0),
                    stream=stream)


def d(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev)


def op(name):
    if name == "lookup":
        return lambda: ctx.bs_draft_lookup(eng.rl_step, eng.slots, k, eng.draft, eng.draft_len,
                                           eng.match_len, stream=stream)
    if name == "target_rows":
        return lambda: ctx.bsx_target_rows(eng.slots, eng.draft, eng.draft_len, k,
                                           eng.target.target_seed, eng.target.mode,
                                           eng.target.nbank, eng.row_index, stream=stream)
    if name == "verify":
        return lambda: ctx.bs_verify_step(eng.slots, bank, eng.row_index, V, eng.draft,
                                          eng.draft_len, k, eng.T, eng.top_p, eng.out_tokens,
                                          eng.out_len, eng.out_acc, stream=stream)
    if name == "commit":
        # commit with out_len = 0 leaves the state unchanged
        return lambda: ctx.bs_commit(eng.slots, eng.out_tokens, zero_len, k, eng.finished,
                                     stream=stream)
    if name == "torch_noop":
        return lambda: scratch.add_(1)
    raise ValueError(name)


scratch = torch.zeros(1, device=dev)
zero_len = torch.zeros(n, dtype=torch.int32, device=dev)


def time_graph(fn, iters=64, reps=20):
    with torch.cuda.stream(stream):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(iters):
                fn()
        g.replay()
        stream.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(reps):
            g.replay()
        e.record(stream)
    e.synchronize()
    return 1000 * s.elapsed_time(e) / (iters * reps)


def begin(live):
    with torch.cuda.stream(stream):
        ctx.bs_draft_pool_put(1, d(h["seq_prompt"]), d(h["seq_off"]), d(h["tokens"]),
                              len(h["tokens"]), stream=stream)
        eng.seal(1)
        ml = h["max_len"].copy()
        ml[live:] = 0  # finished at begin: pos >= max_len
        ml[:live] = 1 << 30
        eng.begin(d(h["uids"].view(np.int64)), d(h["pid"]), d(h["tails"]), d(ml))
        # one real step so drafts / rows exist
        eng.step()
    stream.synchronize()


for live in (0, 1, 8, 256):
    begin(live)
    res = {nm: time_graph(op(nm)) for nm in ("torch_noop", "lookup", "target_rows", "verify", "commit")}
    print(f"live {live:3d}: " + "  ".join(f"{k_} {v:6.2f} us" for k_, v in res.items()))
for live in (1, 8, 32, 256):
    for kind in ("rows", "cluster"):
        ctx.bsx_set_verify_kernel(kind)
        begin(live)
        print(f"live {live:3d} {kind:8s}: verify {time_graph(op('verify')):7.2f} us")
ctx.bsx_set_verify_kernel("auto")
