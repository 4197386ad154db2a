"""f3 measurement: the LM-head GEMM with the fused verify statistics (bs_lm_head_logits) at the
Qwen2.5-7B head (d = 3584, V = 151936), for the row counts of a decoding step (256 rollouts x
1, x 2, x 9 rows), against cuBLAS (torch.matmul, bf16) on the same shapes; then the verify launch
on those logits with and without the fused row statistics (the max pass skipped).

  python scripts/lmhead_bench.py [--iters 10]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_08862_b200 as bs  # noqa: E402


def timed(fn, iters, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for e0, e1 in evs:
        e0.record()
        fn()
        e1.record()
    torch.cuda.synchronize()
    return float(np.median([e0.elapsed_time(e1) for e0, e1 in evs]))


def main(argv=None, quiet=False):
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=3584)
    ap.add_argument("--V", type=int, default=151936)
    ap.add_argument("--rows", default="256,512,2304")
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args(argv)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    d, V = a.d, a.V
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm, tfl = peaks.get("hbm_gbs") or 6650.0, peaks.get("bf16_tflops") or 1645.0
    mult = float(np.float32(3.0 / np.sqrt(d) / 147.8))
    w = torch.empty((V, d), dtype=torch.int16, device=dev)
    bs.bsx_synth_attn_values(w, 22, mult)
    out = {"config": {"d": d, "V": V, "w_gb": V * d * 2 / 1e9}, "gemm": []}
    for rows in (int(x) for x in a.rows.split(",")):
        h = torch.empty((rows, d), dtype=torch.int16, device=dev)
        bs.bsx_synth_attn_values(h, 21, float(np.float32(1.0 / 147.8)))
        lg = torch.empty((rows, V), dtype=torch.int16, device=dev)
        key = torch.empty(rows, dtype=torch.int64, device=dev)
        bad = torch.empty(rows, dtype=torch.int32, device=dev)
        ms = timed(lambda: bs.bs_lm_head_logits(h, w, lg, key, bad), a.iters)
        hb, wb = h.view(torch.bfloat16), w.view(torch.bfloat16)
        ob = torch.empty((rows, V), dtype=torch.bfloat16, device=dev)
        ms_cublas = timed(lambda: torch.matmul(hb, wb.t(), out=ob), a.iters)
        flops = 2.0 * rows * V * d
        bytes_ = V * d * 2 + rows * d * 2 + rows * V * 2
        rec = {"rows": rows, "ms": ms, "tflops": flops / ms / 1e9, "tensor_frac": flops / ms / 1e9 / tfl,
               "hbm_gbs": bytes_ / ms / 1e6, "hbm_frac": bytes_ / ms / 1e6 / hbm,
               "bound": "tensor" if flops / (tfl * 1e12) > bytes_ / (hbm * 1e9) else "hbm",
               "cublas_ms": ms_cublas, "vs_cublas": ms_cublas / ms}
        rec["frac"] = rec["tensor_frac"] if rec["bound"] == "tensor" else rec["hbm_frac"]
        out["gemm"].append(rec)
        del lg, ob
    # verify on LM-head logits (256 rollouts x 9 rows, k = 8), with / without the fused statistics
    n, k = 256, 8
    rows = n * (k + 1)
    h = torch.empty((rows, d), dtype=torch.int16, device=dev)
    bs.bsx_synth_attn_values(h, 23, float(np.float32(1.0 / 147.8)))
    lg, key, bad = bs.bs_lm_head_logits(h, w)
    am = lg.view(torch.bfloat16).float().view(n, k + 1, V).argmax(dim=2).to(torch.int32)
    drafts = am[:, :k].contiguous()
    dlen = torch.full((n,), k, dtype=torch.int32, device=dev)
    slots = torch.arange(n, dtype=torch.int32, device=dev)
    ver = {}
    for use in (False, True):
        ctx = bs.Context(vocab=V, k_max=k, match_max=32, max_rollouts=n, pool_capacity_tokens=16,
                         pool_capacity_seqs=4, seed=5)
        if use:
            ctx.bsx_set_row_stats(key, bad)
        tail = torch.full((n, 32), -1, dtype=torch.int32, device=dev)
        tail[:, -1] = 0
        ctx.bs_rollout_begin(slots, torch.arange(n, dtype=torch.int64, device=dev),
                             torch.zeros(n, dtype=torch.int32, device=dev), tail,
                             torch.full((n,), 1 << 20, dtype=torch.int32, device=dev))
        ot = torch.zeros((n, k + 1), dtype=torch.int32, device=dev)
        ol = torch.zeros(n, dtype=torch.int32, device=dev)
        oa = torch.zeros(n, dtype=torch.int32, device=dev)
        f = lambda ctx=ctx, ot=ot, ol=ol, oa=oa: ctx.bs_verify_step(slots, lg.view(-1), None, V, drafts, dlen, k,  # noqa
                                                                     1.0, 1.0, ot, ol, oa)
        ms = timed(f, a.iters)
        st = ctx.bs_stats_read()
        ver["with_stats" if use else "without_stats"] = {
            "ms": ms, "rows_verified_per_call": int(st[6]) / (a.iters + 3), "tokens": ot.cpu().numpy().tolist()[:2]}
        assert ctx.bs_sync_status() == 0
    ver["speedup"] = ver["without_stats"]["ms"] / ver["with_stats"]["ms"]
    out["verify_on_lm_head_logits"] = ver
    out["peaks"] = {"hbm_gbs": hbm, "bf16_tflops": tfl}
    if not quiet:
        print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    main()
