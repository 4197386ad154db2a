"""Device time of the filtered verify (top-p / top-k, verify_topp_kernel) vs batch size on the
Q7 bank (V=151936): graph-free, CUDA events.
  python scripts/topp_latency.py [--ns 1,8,64] [--k 16] [--top-p 0.95] [--top-k 0]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08862_b200 as bs  # noqa: E402
from workloads import bank_peak  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ns", default="1,8,64")
ap.add_argument("--k", type=int, default=16)
ap.add_argument("--top-p", type=float, default=0.95)
ap.add_argument("--top-k", type=int, default=0)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
V, k, nbank = 151936, a.k, 8192
torch.cuda.set_device(0)
bank = torch.empty((nbank, V), dtype=torch.int16, device="cuda")
bs.bsx_synth_bank(bank, nbank, V, 1, 15.75)
for n in [int(x) for x in a.ns.split(",")]:
    ctx = bs.Context(vocab=V, k_max=k, match_max=32, max_rollouts=n, pool_capacity_tokens=16,
                     pool_capacity_seqs=4, seed=1)
    slots = torch.arange(n, dtype=torch.int32, device="cuda")
    ctx.bs_rollout_begin(slots, torch.arange(n, dtype=torch.int64, device="cuda"),
                         torch.zeros(n, dtype=torch.int32, device="cuda"),
                         torch.zeros((n, 32), dtype=torch.int32, device="cuda"),
                         torch.full((n,), 1 << 30, dtype=torch.int32, device="cuda"))
    rng = np.random.default_rng(n)
    rows = rng.integers(0, nbank, (a.reps, n, k + 1))
    peaks = bank_peak(1, rows.reshape(-1), V).reshape(rows.shape)
    ts = []
    lib = bs.load()
    ph = np.zeros(16, np.uint64)
    timing = hasattr(lib, "bsx_phase_times") and lib.bsx_phase_times(ph.ctypes.data, 1) == 1
    for i in range(a.reps):
        ri = torch.from_numpy(rows[i]).cuda().contiguous()
        dr = torch.from_numpy(peaks[i, :, :k].astype(np.int32)).cuda().contiguous()
        dl = torch.full((n,), k, dtype=torch.int32, device="cuda")
        ot = torch.zeros((n, k + 1), dtype=torch.int32, device="cuda")
        ol = torch.zeros(n, dtype=torch.int32, device="cuda")
        oa = torch.zeros(n, dtype=torch.int32, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.bs_verify_step(slots, bank, ri, V, dr, dl, k, 1.0, a.top_p, ot, ol, oa, top_k=a.top_k)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    st = ctx.bs_stats_read()
    print(f"n={n:4d} top_p={a.top_p} top_k={a.top_k}: median {np.median(ts[2:]):8.1f} us/call, rows verified "
          f"{int(st[6]) / a.reps:.1f}, needed {int(st[7]) / a.reps:.1f}")
    if timing:  # BS_PHASE_TIMING build: thread 0 of every CTA, cycles summed over CTAs and calls
        lib.bsx_phase_times(ph.ctypes.data, 1)
        names = ["claim+clear", "pass 1 max", "pass 2 masses+hist+merge", "filtered pass", "coarse select",
                 "pass 3 keys", "epilogue/sample"]
        tot = float(ph[:15].sum())
        for i, nm in enumerate(names):
            print(f"    {nm:26s} work {100 * float(ph[i]) / tot:5.1f}%  barrier after {100 * float(ph[8 + i]) / tot:5.1f}%")
