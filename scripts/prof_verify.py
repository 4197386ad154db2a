"""Steady-state verify-kernel driver for profiling (ncu / CUDA events): Q7 shape
(V=151936, n=256 rollouts, k=8, all rows live), drafts = the bank rows' peaks (accepted
with p_peak) so the row mix matches the bench.  Prints per-call device time and GB/s."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08862_b200 as bs  # noqa: E402
from workloads import bank_peak  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--V", type=int, default=151936)
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--nbank", type=int, default=8192)
ap.add_argument("--T", type=float, default=1.0)
a = ap.parse_args()
V, n, k = a.V, a.n, a.k
torch.cuda.set_device(0)
bank = torch.empty((a.nbank, V), dtype=torch.int16, device="cuda")
bs.bsx_synth_bank(bank, a.nbank, V, 1, 15.75)
ctx = bs.Context(vocab=V, k_max=k, match_max=32, max_rollouts=n, pool_capacity_tokens=16,
                 pool_capacity_seqs=4, seed=1)
slots = torch.arange(n, dtype=torch.int32, device="cuda")
tail = torch.zeros((n, 32), dtype=torch.int32, device="cuda")
ctx.bs_rollout_begin(slots, torch.arange(n, dtype=torch.int64, device="cuda"),
                     torch.zeros(n, dtype=torch.int32, device="cuda"), tail,
                     torch.full((n,), 1 << 30, dtype=torch.int32, device="cuda"))
rng = np.random.default_rng(0)
rows = rng.integers(0, a.nbank, (a.iters, n, k + 1))
peaks = bank_peak(1, rows.reshape(-1), V).reshape(rows.shape)
ri = torch.from_numpy(rows).cuda()
dr = torch.from_numpy(peaks[:, :, :k].astype(np.int32)).cuda()
dl = torch.full((n,), k, dtype=torch.int32, device="cuda")
ot = torch.zeros((n, k + 1), dtype=torch.int32, device="cuda")
ol = torch.zeros(n, dtype=torch.int32, device="cuda")
oa = torch.zeros(n, dtype=torch.int32, device="cuda")
ts = []
for i in range(a.iters):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    ctx.bs_verify_step(slots, bank, ri[i].contiguous(), V, dr[i].contiguous(), dl, k, a.T, 1.0,
                       ot, ol, oa)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
st = ctx.bs_stats_read()
if os.environ.get("BS_LIB_VARIANT") == "timing":
    import ctypes
    lib = bs.load()
    ph = (ctypes.c_ulonglong * 16)()
    if lib.bsx_phase_times(ph, 1):
        names = ["row start (desc, epilogue slot)", "pass 1 (max) + barrier", "pass 2 (masses)"]
        tot = sum(ph[i] for i in range(len(names)))
        it = max(1, ph[15])
        print(f"phase cycles per row-iteration per CTA (n={ph[15]}):")
        for i, nm in enumerate(names):
            print(f"  {nm:18s} {ph[i] / it:10.0f} cyc  {100 * ph[i] / max(1, tot):5.1f}%")
moved = int(st[6]) * 2 * V
need = int(st[7]) * 2 * V
tot = sum(ts[2:]) / 1e3
frac = (len(ts) - 2) / len(ts)
print(f"verify: median {np.median(ts[2:]):.3f} ms/call, moved {moved * frac / tot / 1e9:.0f} GB/s, "
      f"algorithmic {need * frac / tot / 1e9:.0f} GB/s, AL-ish {int(st[2]) / max(1, int(st[0])):.2f}")
