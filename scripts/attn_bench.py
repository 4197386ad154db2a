"""f2 measurement: the paper's Table 2 setting: batch 128, context 8k, 32 of
the requests speculative with 4 draft tokens (q_len 5), the rest plain decode (q_len 1).

Times (CUDA events, warm-up first, every iteration streams the 2+ GB KV cache: larger than L2)
  unified     one bs_unified_attention launch over the mixed batch          (the paper's 0.380 ms)
  normal      the same batch without speculative queries (all q_len 1)       (0.372 ms)
  batch_split decode requests and speculative requests in two launches       (0.753 + 0.226 ms)
and reports HBM bandwidth on the KV bytes (each request's ctx_len x H_kv x d x 2 (K, V) x 2 B,
plus Q and O) against MEASURED_PEAKS.json.

  python scripts/attn_bench.py [--heads 28,4] [--ctx 8192] [--iters 20]
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

PAGE, D = 64, 128


def main(argv=None, quiet=False):
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--spec", type=int, default=32, help="speculative requests")
    ap.add_argument("--drafts", type=int, default=4)
    ap.add_argument("--ctx", type=int, default=8192)
    ap.add_argument("--heads", default="28,4", help="H_q,H_kv (Qwen2.5-7B 28,4; Qwen3-8B 32,8)")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args(argv)
    H_q, H_kv = (int(x) for x in a.heads.split(","))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    B = a.batch
    ctx = np.full(B, a.ctx, dtype=np.int32)
    q_mixed = np.ones(B, dtype=np.int32)
    q_mixed[np.random.default_rng(0).choice(B, a.spec, replace=False)] = 1 + a.drafts
    npg = (ctx + PAGE - 1) // PAGE
    num_pages = int(npg.sum())
    perm = np.random.default_rng(1).permutation(num_pages).astype(np.int32)
    pt = np.zeros((B, int(npg.max())), dtype=np.int32)
    c = 0
    for b in range(B):
        pt[b, : npg[b]] = perm[c:c + npg[b]]
        c += npg[b]
    mult = float(np.float32(1.0 / 147.8))
    kc = torch.empty((num_pages, H_kv, PAGE, D), dtype=torch.int16, device=dev)
    vc = torch.empty_like(kc)
    bs.bsx_synth_attn_values(kc, 11, mult)
    bs.bsx_synth_attn_values(vc, 12, mult)
    pt_d = torch.from_numpy(pt).to(dev)
    ctx_d = torch.from_numpy(ctx).to(dev)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    hbm = peaks.get("hbm_gbs") or 6650.0

    def q_for(ql):
        q = torch.empty((int(ql.sum()), H_q, D), dtype=torch.int16, device=dev)
        bs.bsx_synth_attn_values(q, 13, mult)
        return q

    def timed(fn):
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.iters)]
        for e0, e1 in evs:
            e0.record()
            fn()
            e1.record()
        torch.cuda.synchronize()
        ts = sorted(e0.elapsed_time(e1) for e0, e1 in evs)
        return float(np.median(ts)), ts[0]

    def kv_bytes(sel):
        return float(ctx[sel].sum()) * H_kv * D * 2 * 2

    res = {"config": {"batch": B, "speculative": a.spec, "drafts": a.drafts, "ctx": a.ctx, "H_q": H_q, "H_kv": H_kv,
                      "head_dim": D, "page": PAGE, "kv_gb": kv_bytes(np.arange(B)) / 1e9,
                      "l2": "every launch streams the whole KV cache (> L2)"}}
    out = {}
    for name, ql in (("unified", q_mixed), ("normal", np.ones(B, dtype=np.int32))):
        q = q_for(ql)
        ws = torch.empty(bs.api.unified_attention_workspace_bytes(ctx, ql, H_q, H_kv), dtype=torch.uint8, device=dev)
        o = torch.empty_like(q)
        fn = lambda q=q, ql=ql, ws=ws, o=o: bs.bs_unified_attention(q, kc, vc, pt_d, ctx_d, ctx, ql, H_kv,  # noqa
                                                                     out=o, workspace=ws)
        med, best = timed(fn)
        gbs = (kv_bytes(np.arange(B)) + 2 * q.numel() * 2) / (med * 1e-3) / 1e9
        out[name] = {"ms": med, "best_ms": best, "hbm_gbs": gbs, "frac": gbs / hbm}
    # batch split: the decode group and the speculative group as two launches
    sel_d, sel_s = np.nonzero(q_mixed == 1)[0], np.nonzero(q_mixed > 1)[0]
    parts = []
    for sel in (sel_d, sel_s):
        ql = q_mixed[sel]
        q = q_for(ql)
        ws = torch.empty(bs.api.unified_attention_workspace_bytes(ctx[sel], ql, H_q, H_kv), dtype=torch.uint8,
                         device=dev)
        parts.append((q, ql, torch.from_numpy(np.ascontiguousarray(pt[sel])).to(dev),
                      torch.from_numpy(np.ascontiguousarray(ctx[sel])).to(dev), ctx[sel], ws, torch.empty_like(q)))

    def split():
        for q, ql, p_, c_, ch, ws, o in parts:
            bs.bs_unified_attention(q, kc, vc, p_, c_, ch, ql, H_kv, out=o, workspace=ws)

    med, best = timed(split)
    out["batch_split"] = {"ms": med, "best_ms": best}
    res.update(out)
    res["unified_over_normal"] = out["unified"]["ms"] / out["normal"]["ms"]
    res["paper"] = {"normal_ms": 0.372, "split_prefill_ms": 0.753, "split_decode_ms": 0.226, "unified_ms": 0.380,
                    "note": "P:229-231, unstated GPU/model: context only"}
    res["peak_gbs"] = hbm
    if not quiet:
        print(json.dumps(res), flush=True)
    return res


if __name__ == "__main__":
    main()
