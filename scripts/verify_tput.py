"""Raw throughput / latency of the verify launch on the Q7 bank with (almost) certain
acceptance: beta large, drafts = the rows' peaks, so every row of every rollout is needed.
  BS_FORCE_EAGER=1 python scripts/verify_tput.py --ns 256 --beta 40"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08862_b200 as bs  # noqa: E402
from workloads import bank_peak  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ns", default="1,8,64,256")
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--reps", type=int, default=16)
ap.add_argument("--beta", type=float, default=40.0)
ap.add_argument("--kind", type=int, default=0)
a = ap.parse_args()
V, k, nbank = 151936, a.k, 8192
torch.cuda.set_device(0)
bank = torch.empty((nbank, V), dtype=torch.int16, device="cuda")
bs.bsx_synth_bank(bank, nbank, V, 1, a.beta)
st = torch.cuda.Stream()
for n in [int(x) for x in a.ns.split(",")]:
    ctx = bs.Context(vocab=V, k_max=k, match_max=32, max_rollouts=n, pool_capacity_tokens=16,
                     pool_capacity_seqs=4, seed=1)
    if a.kind:
        ctx.bsx_set_verify_kernel(a.kind)
    slots = torch.arange(n, dtype=torch.int32, device="cuda")
    ctx.bs_rollout_begin(slots, torch.arange(n, dtype=torch.int64, device="cuda"),
                         torch.zeros(n, dtype=torch.int32, device="cuda"),
                         torch.zeros((n, 32), dtype=torch.int32, device="cuda"),
                         torch.full((n,), 1 << 30, dtype=torch.int32, device="cuda"))
    rng = np.random.default_rng(n)
    rows = rng.integers(0, nbank, (a.reps, n, k + 1))
    peaks = bank_peak(1, rows.reshape(-1), V).reshape(rows.shape)
    ri = [torch.from_numpy(rows[i]).cuda().contiguous() for i in range(a.reps)]
    dr = [torch.from_numpy(peaks[i, :, :k].astype(np.int32)).cuda().contiguous() for i in range(a.reps)]
    dl = torch.full((n,), k, dtype=torch.int32, device="cuda")
    ot = torch.zeros((n, k + 1), dtype=torch.int32, device="cuda")
    ol = torch.zeros(n, dtype=torch.int32, device="cuda")
    oa = torch.zeros(n, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        for i in range(3):
            ctx.bs_verify_step(slots, bank, ri[i], V, dr[i], dl, k, 1.0, 1.0, ot, ol, oa, stream=st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for i in range(a.reps):
                ctx.bs_verify_step(slots, bank, ri[i], V, dr[i], dl, k, 1.0, 1.0, ot, ol, oa, stream=st)
        g.replay()
        st.synchronize()
        s0 = ctx.bs_stats_read()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.replay()
        e1.record(st)
        st.synchronize()
        s1 = ctx.bs_stats_read()
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    rv = (int(s1[6]) - int(s0[6])) / a.reps
    rn = (int(s1[7]) - int(s0[7])) / a.reps
    acc = (int(s1[4]) - int(s0[4])) / a.reps
    print(f"n={n:4d}: {us:7.1f} us/call  rows verified {rv:6.1f} needed {rn:6.1f} accepted {acc:6.1f} "
          f"algorithmic {rn * 2 * V / us / 1e3:6.0f} GB/s  moved {rv * 2 * V / us / 1e3:6.0f} GB/s", flush=True)
    del ctx
