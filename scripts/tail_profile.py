"""Where does an RL step's time go?  Runs the bench's q7 RL step through the engine and
times every graph chunk (64 decode iterations) with CUDA events, next to the number of live
rollouts at the chunk's end and the device time of the verify calls inside it.
  python scripts/tail_profile.py [--chunk 64]"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2605_08862_b200 as bs  # noqa: E402
from paper_2605_08862_b200.engine import RolloutEngine, Target  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--chunk", type=int, default=64)
ap.add_argument("--config", default="q7")
ap.add_argument("--no-events", action="store_true", help="time whole chunks only (no event nodes)")
ap.add_argument("--separate", action="store_true", help="lookup kernel + bs_verify_commit (default: fused lookup)")
a = ap.parse_args()
cfg = bench.CONFIGS[a.config]
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


chunk = a.chunk
# ev[i][0..4]: before lookup, target rows, verify, commit, after commit
ev = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(5)] for _ in range(chunk)]
OPS = ["lookup", "target_rows", "verify", "commit"]  # (fused: lookup inside verify)
import time as _time  # noqa: E402

for rl in (1, 2):
    t0 = _time.perf_counter()
    with torch.cuda.stream(stream):
        ctx.bs_draft_pool_put(rl, d(h["seq_prompt"]), d(h["seq_off"]), d(h["tokens"]),
                              len(h["tokens"]), stream=stream)
        stream.synchronize()
        t1 = _time.perf_counter()
        eng.seal(rl)
        stream.synchronize()
        t2 = _time.perf_counter()
        eng.begin(d(h["uids"].view(np.int64)), d(h["pid"]), d(h["tails"]), d(h["max_len"]))
    rec = not a.no_events
    with torch.cuda.stream(stream):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(chunk):
                if rec:
                    ev[i][0].record(stream)
                if a.separate:  # the lookup kernel (else: fused into the previous verify launch)
                    ctx.bs_draft_lookup(eng.rl_step, eng.slots, k, eng.draft, eng.draft_len,
                                        eng.match_len, stream=stream)
                if rec:
                    ev[i][1].record(stream)
                ctx.bsx_target_rows(eng.slots, eng.draft, eng.draft_len, k, eng.target.target_seed,
                                    eng.target.mode, eng.target.nbank, eng.row_index, stream=stream)
                if rec:
                    ev[i][2].record(stream)
                if a.separate:
                    ctx.bs_verify_commit(eng.slots, bank, eng.row_index, V, eng.draft, eng.draft_len, k,
                                         eng.T, eng.top_p, eng.out_tokens, eng.out_len, eng.out_acc,
                                         eng.finished, stream=stream)
                else:
                    ctx.bs_verify_commit_lookup(eng.rl_step, eng.slots, bank, eng.row_index, V, eng.draft,
                                                eng.draft_len, k, eng.T, eng.top_p, eng.out_tokens,
                                                eng.out_len, eng.out_acc, eng.finished, eng.match_len,
                                                stream=stream)
                if rec:
                    ev[i][3].record(stream)
                pass
                if rec:
                    ev[i][4].record(stream)
    stream.synchronize()
    t3 = _time.perf_counter()
    rows = []
    cs, ce = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    while True:
        with torch.cuda.stream(stream):
            cs.record(stream)
            g.replay()
            ce.record(stream)
            live = int((~eng.finished.bool()).sum().item())
        tot = cs.elapsed_time(ce)
        per = ([sum(ev[i][o].elapsed_time(ev[i][o + 1]) for i in range(chunk)) for o in range(4)]
               if rec else [0.0] * 4)
        rows.append([live, tot] + per)
        if live == 0:
            break
    t4 = _time.perf_counter()
    if rl == 2:
        print(f"host wall: put {1e3 * (t1 - t0):.1f} ms, seal {1e3 * (t2 - t1):.1f} ms, "
              f"begin+capture {1e3 * (t3 - t2):.1f} ms, decode loop {1e3 * (t4 - t3):.1f} ms")
        arr = np.array(rows)
        T = arr[:, 1].sum()
        print(f"chunks {len(rows)}, total {T:.1f} ms; " + ", ".join(
            f"{o} {arr[:, 2 + i].sum():.1f} ms" for i, o in enumerate(OPS)))
        for lo, hi in [(129, 256), (33, 128), (9, 32), (3, 8), (2, 2), (1, 1), (0, 0)]:
            m = (arr[:, 0] >= lo) & (arr[:, 0] <= hi)
            if m.any():
                print(f"live at chunk end in [{lo:3d},{hi:3d}]: {m.sum():5d} chunks, "
                      f"{arr[m, 1].sum():8.1f} ms ({100 * arr[m, 1].sum() / T:4.1f}%), "
                      f"{1000 * arr[m, 1].mean() / chunk:6.1f} us/iter: " + " ".join(
                          f"{o} {1000 * arr[m, 2 + i].mean() / chunk:5.1f}" for i, o in enumerate(OPS)))
        st = eng.stats(reset=True)
        print({k_: st[k_] for k_ in ("acceptance_length", "acceptance_rate", "tokens", "decode_steps")})
