"""Standalone draft-lookup driver (K1 `lookup_kernel`) on the bench's Q7 state, for ncu:
the L2 hit rate of the index probes (north_star: "L2 hit rate for the draft index").

Q7 inputs of RL step 0 (16 prompts x 16 pools, ~0.7 M pool tokens), 256 rollouts begun and
advanced by a few fused decoding steps so their tails are mid-response, then `--iters`
bs_draft_lookup calls on the same state (k = 8).  Prints per-call device time and the index
size.  Profile with
  ncu --set full -k regex:lookup_kernel -c 3 python scripts/prof_lookup.py
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2605_08862_b200 as bs  # noqa: E402
from paper_2605_08862_b200.engine import TARGET_MODES, RolloutEngine, Target  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--advance", type=int, default=200, help="decoding steps before the lookups")
ap.add_argument("--decode", action="store_true",
                help="after the advance, run --iters decoding steps with the lookup as its own kernel "
                     "(lookup -> target rows -> verify+commit), so each lookup sees the L2 state a "
                     "decoding step leaves (profile with --cache-control none)")
a = ap.parse_args()
cfg = bench.CONFIGS["q7"]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
h = bench.make_step_inputs(cfg, 0, 0, 1)
V, k, n = cfg["V"], cfg["k"], len(h["pid"])
spec = h["spec"]
bank = torch.empty((cfg["nbank"], V), dtype=torch.int16, device=dev)
bs.bsx_synth_bank(bank, cfg["nbank"], V, spec.bank_seed, spec.beta)
ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=cfg["M"], max_rollouts=n,
                 pool_capacity_tokens=len(h["tokens"]) + 16, pool_capacity_seqs=len(h["seq_prompt"]) + 4,
                 device=0, seed=0x5EED)
eng = RolloutEngine(ctx, n, k, cfg["T"], cfg["top_p"],
                    Target(bank, cfg["nbank"], spec.target_seed, TARGET_MODES[spec.mode]))
d = {key: torch.from_numpy(np.ascontiguousarray(v if key != "uids" else v.view(np.int64))).to(dev)
     for key, v in dict(sp=h["seq_prompt"], off=h["seq_off"], tok=h["tokens"], pid=h["pid"], tails=h["tails"],
                         uids=h["uids"], ml=h["max_len"]).items()}
eng.put_pools(1, d["sp"], d["off"], d["tok"])
eng.seal(1)
eng.begin(d["uids"], d["pid"], d["tails"], d["ml"])
with torch.cuda.stream(eng.stream):
    for _ in range(a.advance):
        eng.step()
torch.cuda.synchronize()
if a.decode:
    eng.fuse_lookup = False  # bs_verify_commit + a separate bs_draft_lookup per step
    with torch.cuda.stream(eng.stream):
        for _ in range(a.iters):
            eng.step()
    torch.cuda.synchronize()
    assert ctx.bs_sync_status() == 0
    print("decode mode: ran", a.iters, "steps with standalone lookups")
    sys.exit(0)
def timed_calls(fn):
    out = []
    for _ in range(a.iters):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(eng.stream):
            s.record(eng.stream)
            fn()
            e.record(eng.stream)
        torch.cuda.synchronize()
        out.append(s.elapsed_time(e) * 1e3)
    return out


# the n-gram linear-scan drafter (f4) on the same state, for the per-call comparison
tn = timed_calls(lambda: ctx.bs_draft_lookup_ngram(1, eng.slots, k, 1, 32, eng.draft, eng.draft_len, eng.match_len,
                                                    stream=eng.stream))
dl_ng = eng.draft_len.cpu().numpy().copy()
ts = timed_calls(lambda: ctx.bs_draft_lookup(1, eng.slots, k, eng.draft, eng.draft_len, eng.match_len,
                                             stream=eng.stream))
assert ctx.bs_sync_status() == 0
ml = eng.match_len.cpu().numpy()
dl = eng.draft_len.cpu().numpy()
print(f"lookup: {n} rollouts, pool {len(h['tokens'])} tokens, median {np.median(ts[2:]):.1f} us/call, "
      f"mean anchor {ml.mean():.1f}, mean draft {dl.mean():.2f}")
print(f"ngram drafter: median {np.median(tn[2:]):.1f} us/call, mean draft {dl_ng.mean():.2f}")
