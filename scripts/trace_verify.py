"""Latency anatomy of the cluster verify kernel from its event trace (BS_TRACE build).
  python -m paper_2605_08862_b200.build --trace
  BS_LIB_VARIANT=trace python scripts/trace_verify.py [--n 256] [--k 8] [--accept peak|none]
Runs a few steady-state bs_verify_step calls (Q7 shapes: bank rows, drafts = the rows' peaks,
accepted with p_peak), then prints, per row stage, the median / p90 duration in us:
claim, claim->TMA issue, TMA issue->data landed (max start), max, max exchange, masses,
sum exchange, epilogue; and the kernel span."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BS_LIB_VARIANT", "trace")
import paper_2605_08862_b200 as bs  # noqa: E402
from workloads import bank_peak  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--V", type=int, default=151936)
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--nbank", type=int, default=8192)
ap.add_argument("--bench", type=int, default=0, help="trace the bench q7 loop after this many decode steps")
ap.add_argument("--live", type=int, default=0, help="synthetic: only this many live rollouts (rest finished)")
a = ap.parse_args()
V, n, k = a.V, a.n, a.k
lib = bs.load()
lib.bsx_trace_read.restype = ctypes.c_int
lib.bsx_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
torch.cuda.set_device(0)
buf = np.zeros((1 << 20, 4), dtype=np.uint32)
res = []
if a.bench:
    import bench
    from paper_2605_08862_b200.engine import RolloutEngine, Target
    cfg = bench.CONFIGS["q7"]
    V, k = cfg["V"], cfg["k"]
    h = bench.make_step_inputs(cfg, 0, 0, 1)
    n = cfg["prompts"] * cfg["G"]
    ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=cfg["M"], max_rollouts=n,
                     pool_capacity_tokens=len(h["tokens"]) + 16, pool_capacity_seqs=len(h["seq_prompt"]) + 4,
                     seed=0x5EED)
    spec = h["spec"]
    bank = torch.empty((cfg["nbank"], V), dtype=torch.int16, device="cuda")
    bs.bsx_synth_bank(bank, cfg["nbank"], V, spec.bank_seed, spec.beta)
    eng = RolloutEngine(ctx, n, k, cfg["T"], cfg["top_p"], Target(bank, cfg["nbank"], spec.target_seed, 0))
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    eng.put_pools(1, d(h["seq_prompt"]), d(h["seq_off"]), d(h["tokens"]))
    eng.seal(1)
    eng.begin(d(h["uids"].view(np.int64)), d(h["pid"]), d(h["tails"]), d(h["max_len"]))
    for i in range(a.bench + a.iters):
        c, t_ = ctx, eng.target
        c.bs_draft_lookup(eng.rl_step, eng.slots, k, eng.draft, eng.draft_len, eng.match_len)
        c.bsx_target_rows(eng.slots, eng.draft, eng.draft_len, k, t_.target_seed, t_.mode, t_.nbank, eng.row_index)
        torch.cuda.synchronize()
        lib.bsx_trace_read(buf.ctypes.data, 1 << 20, 1)
        st0 = ctx.bs_stats_read()
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record()
        c.bs_verify_step(eng.slots, bank, eng.row_index, V, eng.draft, eng.draft_len, k, eng.T, eng.top_p,
                         eng.out_tokens, eng.out_len, eng.out_acc)
        e_.record()
        torch.cuda.synchronize()
        st1 = ctx.bs_stats_read()
        m = lib.bsx_trace_read(buf.ctypes.data, 1 << 20, 1)
        c.bs_commit(eng.slots, eng.out_tokens, eng.out_len, k, eng.finished)
        if i >= a.bench:
            res.append((s_.elapsed_time(e_), m, buf[:m].copy(), int(st1[6] - st0[6]), int(st1[7] - st0[7])))
    n = int((~eng.finished.bool()).sum().item())
else:
    bank = torch.empty((a.nbank, V), dtype=torch.int16, device="cuda")
    bs.bsx_synth_bank(bank, a.nbank, V, 1, 13.5)
    ctx = bs.Context(vocab=V, k_max=k, match_max=32, max_rollouts=n, pool_capacity_tokens=16,
                     pool_capacity_seqs=4, seed=1)
    slots = torch.arange(n, dtype=torch.int32, device="cuda")
    mlen = torch.full((n,), 1 << 30, dtype=torch.int32, device="cuda")
    if a.live:
        mlen[a.live:] = 0
    ctx.bs_rollout_begin(slots, torch.arange(n, dtype=torch.int64, device="cuda"),
                         torch.zeros(n, dtype=torch.int32, device="cuda"),
                         torch.zeros((n, 32), dtype=torch.int32, device="cuda"), mlen)
    rng = np.random.default_rng(0)
    rows = rng.integers(0, a.nbank, (a.iters, n, k + 1))
    peaks = bank_peak(1, rows.reshape(-1), V).reshape(rows.shape)
    ri = torch.from_numpy(rows).cuda()
    dr = torch.from_numpy(peaks[:, :, :k].astype(np.int32)).cuda()
    dl = torch.full((n,), k, dtype=torch.int32, device="cuda")
    ot = torch.zeros((n, k + 1), dtype=torch.int32, device="cuda")
    ol = torch.zeros(n, dtype=torch.int32, device="cuda")
    oa = torch.zeros(n, dtype=torch.int32, device="cuda")
    for i in range(a.iters):
        lib.bsx_trace_read(buf.ctypes.data, 1 << 20, 1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st0 = ctx.bs_stats_read()
        s.record()
        ctx.bs_verify_step(slots, bank, ri[i].contiguous(), V, dr[i].contiguous(), dl, k, 1.0, 1.0, ot, ol, oa)
        e.record()
        torch.cuda.synchronize()
        st1 = ctx.bs_stats_read()
        m = lib.bsx_trace_read(buf.ctypes.data, 1 << 20, 1)
        res.append((s.elapsed_time(e), m, buf[:m].copy(), int(st1[6] - st0[6]), int(st1[7] - st0[7])))

names = ["claim0", "claim1", "tma", "max0", "max1", "mass0", "mass1", "epi0", "epi1", "end", "fin", "spins", "sc",
         "sqpop", "iter", "massl", "start", "go", "planned", "pdesc", "post", "loop", "bcast"]
ms, m, ev, rv, rn = res[-1]
if os.environ.get("TRACE_SAVE"):
    np.save(os.environ["TRACE_SAVE"], ev)
blk = ev[:, 0] & 0xFFFF
typ = (ev[:, 0] >> 16) & 0xFF
jj = ev[:, 0] >> 24
seq = ev[:, 1] & 0xFFFF
bb = ev[:, 1] >> 16
t = (ev[:, 2].astype(np.uint64) | (ev[:, 3].astype(np.uint64) << np.uint64(32))).astype(np.int64)
t0 = t.min()
t = (t - t0) / 1e3  # us
print(f"n={n} k={k}: last call {ms * 1e3:.1f} us (events), rows verified {rv}, needed {rn}, "
      f"trace events {m}, kernel span {t[typ == 9].max():.1f} us")
key = {}
for i in range(m):
    key.setdefault((int(typ[i]), int(blk[i]), int(seq[i])), []).append(t[i])


def stage(a_, b_, leader_only=False, label=""):
    d = []
    for (ty, bl, sq), ts in key.items():
        if ty != a_ or (leader_only and bl % 8):
            continue
        o = key.get((b_, bl, sq))
        if o:
            d.append(o[-1] - ts[0])
    d = np.array(d)
    if len(d):
        print(f"  {label:28s} n={len(d):5d} median {np.median(d):6.2f}  p90 {np.percentile(d, 90):6.2f}  "
              f"max {d.max():6.2f} us")


stage(0, 1, True, "claim (leader)")
stage(2, 3, False, "TMA issue -> max start")
stage(3, 4, False, "max (slice)")
stage(4, 5, False, "max publish -> mass start")
stage(5, 6, False, "masses (slice)")
stage(6, 7, False, "mass end -> epilogue start")
stage(7, 8, False, "epilogue")
# claim end (leader, row r) -> TMA issue (leader, row r)
d = []
for (ty, bl, sq), ts in key.items():
    if ty == 1 and bl % 8 == 0:
        o = key.get((2, bl, sq))
        if o:
            d.append(o[0] - ts[-1])
if d:
    d = np.array(d)
    print(f"  {'claim end -> TMA issue':28s} n={len(d):5d} median {np.median(d):6.2f}  p90 {np.percentile(d, 90):6.2f}")
# rows per cluster and busy fraction
lead = (typ == 2) & (blk % 8 == 0)
print(f"  rows per cluster: mean {lead.sum() / max(1, len(set(blk[blk % 8 == 0]))):.1f}; "
      f"first TMA at {t[lead].min():.1f} us, last epilogue end {t[typ == 8].max():.1f} us")
print("all calls (us):", " ".join(f"{r[0] * 1e3:.1f}" for r in res))
if os.environ.get("TRACE_TAIL"):
    endt = {int(bl): float(tt) for bl, tt, ty in zip(blk, t, typ) if ty == 9}
    for bl in sorted(endt, key=lambda x: -endt[x])[:6]:
        evs = sorted((float(tt), names[int(ty)], int(sq), int(b_), int(j_)) for tt, ty, sq, b_, j_, bk in
                     zip(t, typ, seq, bb, jj, blk) if bk == bl)
        print(f"block {bl} END {endt[bl]:.1f}: last events", [(f"{e[0]:.1f}", e[1], e[2], e[3], e[4]) for e in evs[-8:]])
    c1 = [(float(tt), int(b_)) for tt, ty, b_, bk in zip(t, typ, bb, blk) if ty == 1]
    ends = sorted(tt for tt, b_ in c1 if b_ == 0xFFFF)
    print("END claims (b=-1) at:", [f"{x:.1f}" for x in ends[:5]], "...", [f"{x:.1f}" for x in ends[-5:]])
    fins = sorted(float(tt) for tt, ty in zip(t, typ) if ty == 10)
    print(f"finalizes: {len(fins)}, last at", [f"{x:.1f}" for x in fins[-4:]])
    sp = [(float(tt), int(sq)) for tt, ty, sq in zip(t, typ, seq) if ty == 11]
    print("spin counts at END:", sorted(x[1] for x in sp)[:5], sorted(x[1] for x in sp)[-5:])
    lastc = max((float(tt), int(bk)) for tt, ty, bk in zip(t, typ, blk) if ty == 1)
    bl = lastc[1]
    evs = sorted((float(tt), names[int(ty)], int(sq), int(b_), int(j_)) for tt, ty, sq, b_, j_, bk in
                 zip(t, typ, seq, bb, jj, blk) if bk == bl)
    print(f"leader block {bl} full event list:")
    for e in evs:
        print("   ", f"{e[0]:8.1f}", e[1], e[2], e[3], e[4])
if os.environ.get("TRACE_ALL"):
    evs = sorted((float(tt), int(bk), names[int(ty)], int(sq), int(b_), int(j_)) for tt, ty, sq, b_, j_, bk in
                 zip(t, typ, seq, bb, jj, blk) if ty in (0, 1, 2, 7, 8, 9, 10, 11) and (bk % 8 == 0 or ty in (7, 8, 10)))
    for e in evs:
        if e[2] in ("epi0", "epi1") and e[4] == 0 and e[5] == 0 and e[2] != "fin":
            pass
        print("   ", f"{e[0]:8.2f}", *e[1:])
if os.environ.get("TRACE_CL"):
    c = int(os.environ["TRACE_CL"])
    evs = sorted((float(tt), int(bk), names[int(ty)], int(sq), int(b_), int(j_)) for tt, ty, sq, b_, j_, bk in
                 zip(t, typ, seq, bb, jj, blk) if bk == 8 * c)
    for e in evs:
        print("   ", f"{e[0]:8.2f}", *e[1:])
if os.environ.get("TRACE_FLIGHT"):
    # rows in flight over time (leader TMA issue -> leader epilogue end) and claim sources
    starts = {}
    for tt, ty, sq, bk in zip(t, typ, seq, blk):
        if bk % 8 == 0 and ty == 2:
            starts[(int(bk), int(sq) & 0xFFF)] = float(tt)
    iv = []
    for tt, ty, sq, bk in zip(t, typ, seq, blk):
        if bk % 8 == 0 and ty == 8 and (int(bk), int(sq) & 0xFFF) in starts:
            iv.append((starts[(int(bk), int(sq) & 0xFFF)], float(tt)))
    span = t[typ == 9].max()
    for x in np.arange(0, span, 10.0):
        inf = sum(1 for s_, e_ in iv if s_ <= x + 5 < e_)
        src = [int(sq) >> 12 for tt, ty, sq, bk in zip(t, typ, seq, blk) if ty == 1 and x <= tt < x + 10 and int(bb[0]) >= 0]
        cl = [(int(sq) >> 12) for tt, ty, sq, bk, b_ in zip(t, typ, seq, blk, bb) if ty == 1 and x <= tt < x + 10 and b_ != 0xFFFF]
        print(f"  t={x:6.1f}: in flight {inf:3d}; claims ready {cl.count(1)} static {cl.count(2)} spec {cl.count(3)}")
    for tt, ty, sq, b_, j_ in zip(t, typ, seq, bb, jj):
        if ty == 12:
            print(f"  {'SQ' if j_ == 0 else 'RQ'} head {sq} resv {b_}")
    pops = sorted((float(tt), int(sq), int(b_) & 0xFF, int(b_) >> 8, int(j_)) for tt, ty, sq, b_, j_ in zip(t, typ, seq, bb, jj) if ty == 13)
    print(f"  SQ pops: {len(pops)}")
    for p_ in pops[:40]:
        print(f"    t={p_[0]:7.2f} head {p_[1]} L {p_[2]} nw {p_[3]} ok {p_[4] >> 1} live {p_[4] & 1}")
    its = sorted((float(tt), int(bk), int(sq), int(b_), int(j_)) for tt, ty, sq, b_, j_, bk in zip(t, typ, seq, bb, jj, blk) if ty == 14 and bk == 40)
    print(f"  claim iterations of block 40: {len(its)}")
    for p_ in its[:60]:
        print(f"    t={p_[0]:7.2f} spin {p_[2]} b {p_[3]} src {p_[4]}")
if os.environ.get("TRACE_MASS"):
    # per (block, row): spread of mass-warp start times and loop end times
    st_, en_ = {}, {}
    for tt, ty, sq, b_, bk in zip(t, typ, seq, bb, blk):
        if ty == 5:
            st_.setdefault((int(bk), int(sq)), []).append(float(tt))
        if ty == 15:
            en_.setdefault((int(bk), int(sq)), []).append(float(tt))
    sp, ln, lo = [], [], []
    for key_, v in st_.items():
        if key_ in en_ and len(v) == 8 and len(en_[key_]) == 8:
            sp.append(max(v) - min(v))
            ln.append(max(en_[key_]) - min(v))
            lo.append(min(en_[key_]) - min(v))
    print(f"  mass warps: start spread median {np.median(sp):.2f} us; first loop end {np.median(lo):.2f}; "
          f"last loop end {np.median(ln):.2f} us (from first start), rows {len(sp)}")
    cyc = [int(j_) * 64 for tt, ty, j_ in zip(t, typ, jj) if ty == 15]
    print(f"  mass loop cycles per warp: median {np.median(cyc):.0f} p90 {np.percentile(cyc, 90):.0f} (x64 quantized)")
    # which warps finish their mass loop last (per-warp mean lateness vs the row's first finish)
    fin_w = collections.defaultdict(list) if False else {}
    per_row = {}
    for tt, ty, b_, bk, sq in zip(t, typ, bb, blk, seq):
        if ty == 15:
            per_row.setdefault((int(bk), int(sq)), {})[int(b_)] = float(tt)
    late = np.zeros(8); cnt = np.zeros(8)
    for key_, d_ in per_row.items():
        if len(d_) == 8:
            m0 = min(d_.values())
            for w_, tt in d_.items():
                late[w_] += tt - m0
                cnt[w_] += 1
    print("  mass loop lateness by warp (us):", " ".join(f"w{w_}:{late[w_] / max(1, cnt[w_]):.2f}" for w_ in range(8)))

if os.environ.get("TRACE_PHASES"):
    def tmin(ty):
        v = t[typ == ty]
        return (v.min(), v.max()) if len(v) else (float("nan"), float("nan"))
    for ty, nm in [(16, "CTA start"), (17, "past pdl_wait"), (18, "rollout planned"), (1, "claim end"),
                   (2, "TMA issue"), (8, "epilogue end"), (10, "finalize"), (9, "CTA exit")]:
        lo, hi = tmin(ty)
        print(f"  {nm:16s} first {lo:7.2f}  last {hi:7.2f} us")
if os.environ.get("TRACE_SM"):
    sm = {int(bk): int(b_) for ty, bk, b_ in zip(typ, blk, bb) if ty == 16}
    from collections import Counter
    occ = Counter(sm.values())
    ncl = max(sm) // 8 + 1
    print(f"  CTAs {len(sm)}, SMs used {len(occ)}, doubly occupied {sum(1 for v in occ.values() if v > 1)}")
    for c in range(min(ncl, 12)):
        sms = [sm.get(8 * c + r, -1) for r in range(8)]
        partners = sorted({bk // 8 for bk, s_ in sm.items() if s_ in sms and bk // 8 != c})
        print(f"  cluster {c:2d}: SMs {sms} shares with clusters {partners}")
if os.environ.get("TRACE_ROWS"):
    # per working cluster (leader): stage times of its row(s)
    for bl in sorted(set(int(x) for x in blk[(typ == 2)])):
        if bl % 8:
            continue
        ev_ = sorted((float(tt), names[int(ty)], int(sq) & 0xFFF, int(b_), int(j_)) for tt, ty, sq, b_, j_, bk in
                     zip(t, typ, seq, bb, jj, blk) if bk // 8 == bl // 8 and ty in (2, 3, 4, 5, 6, 7, 8, 10))
        print(f"  cluster {bl // 8}:", " ".join(f"{e[1]}@{e[0]:.1f}" for e in ev_ if e[1] in ('tma', 'epi1', 'fin') or True)[:600])
if os.environ.get("TRACE_BUSY"):
    # mass-warp busy fraction per CTA over time windows (warp 0's MASS0 -> MASSL)
    m0 = {}
    busy = []
    for tt, ty, sq, b_, bk in zip(t, typ, seq, bb, blk):
        if ty == 5 and int(b_) == 0:
            m0[(int(bk), int(sq))] = float(tt)
        if ty == 15 and int(b_) == 0 and (int(bk), int(sq)) in m0:
            busy.append((m0[(int(bk), int(sq))], float(tt)))
    span = t[typ == 9].max()
    ncta = len(set(int(x) for x in blk))
    for x in np.arange(0, span, 10.0):
        occ = sum(max(0.0, min(e_, x + 10) - max(s_, x)) for s_, e_ in busy)
        print(f"  t={x:6.1f}: mass warps busy {100 * occ / (10.0 * ncta):5.1f}% of CTA time")
if os.environ.get("TRACE_GAPS"):
    # per leader CTA: consecutive rows i, i+1 -> mass idle gap and what row i+1 waited for
    ev = {}
    for tt, ty, sq, b_, bk in zip(t, typ, seq, bb, blk):
        if int(bk) % 8:
            continue
        k_ = (int(ty), int(bk), int(sq) & 0xFFF)
        if int(ty) in (5, 15) and int(b_) != 0:
            continue  # warp 0 only for mass events
        ev.setdefault(k_, float(tt))
    gaps, wmax, wtma, wclaim, wc0, wcd, wbc, wpd, wpt = [], [], [], [], [], [], [], [], []
    for (ty, bk, sq), tt in ev.items():
        if ty != 6:  # mass1 of row sq
            continue
        nxt = ev.get((5, bk, sq + 1))
        if nxt is None:
            continue
        gaps.append(nxt - tt)
        mx1 = ev.get((4, bk, sq + 1))
        tma1 = ev.get((2, bk, sq + 1))
        prev_end = ev.get((6, bk, sq - 1))
        cl = ev.get((1, bk, sq + 1))
        c0 = ev.get((0, bk, sq + 1))
        if c0 is not None and prev_end is not None:
            wc0.append(c0 - prev_end)
            if cl is not None:
                wcd.append(cl - c0)
            if tma1 is not None and cl is not None:
                wbc.append(tma1 - cl)
            pd = ev.get((19, bk, sq + 1))
            if pd is not None and cl is not None and tma1 is not None:
                wpd.append(pd - cl)
                wpt.append(tma1 - pd)
        if mx1 is not None:
            wmax.append(mx1 - tt)
        if tma1 is not None and prev_end is not None:
            wtma.append(tma1 - prev_end)
        if cl is not None and prev_end is not None:
            wclaim.append(cl - prev_end)
    q = lambda v: f"median {np.median(v):6.2f} p75 {np.percentile(v, 75):6.2f} p90 {np.percentile(v, 90):6.2f}" if v else "-"
    print("  mass idle gap (next mass0 - mass1):", q(gaps))
    print("  next max1 - mass1 (>0: waiting for max):", q(wmax))
    print("  next TMA issue - previous-row mass1 (buffer free):", q(wtma))
    print("  next claim end - previous-row mass1:", q(wclaim))
    print("  next claim start (past issued / dempty waits) - previous-row mass1:", q(wc0))
    print("  claim start -> claim end:", q(wcd))
    print("  claim end -> TMA issue:", q(wbc))
    print("  claim end -> producer has the descriptor:", q(wpd))
    print("  producer has the descriptor -> TMA issue (buffer wait):", q(wpt))
if os.environ.get("TRACE_CLAIMS"):
    c0, c1 = {}, {}
    for tt, ty, sq, b_, bk in zip(t, typ, seq, bb, blk):
        if int(bk) % 8:
            continue
        key_ = (int(bk), int(sq) & 0xFFF)
        if ty == 0:
            c0.setdefault(key_, float(tt))
        if ty == 1:
            c1[key_] = (float(tt), int(sq) >> 12, int(b_))
    bysrc = {}
    for key_, (tt, src, b_) in c1.items():
        if key_ in c0 and b_ != 0xFFFF:
            bysrc.setdefault(src, []).append(tt - c0[key_])
    for src, v in sorted(bysrc.items()):
        print(f"  claim duration src {src}: n={len(v)} median {np.median(v):.2f} p75 {np.percentile(v, 75):.2f} p90 {np.percentile(v, 90):.2f} us")
if os.environ.get("TRACE_CHAIN"):
    # the rollouts finalized last: per row, claim end / TMA issue / epilogue end (leader) and source
    fin = sorted(((float(tt), int(b_), int(j_)) for tt, ty, b_, j_ in zip(t, typ, bb, jj) if ty == 10), reverse=True)
    rows = {}
    for tt, ty, sq, b_, j_, bk in zip(t, typ, seq, bb, jj, blk):
        if int(bk) % 8:
            continue
        if ty == 1 and int(b_) != 0xFFFF:
            rows.setdefault((int(b_), int(j_)), {})["claim"] = (float(tt), int(sq) >> 12, int(bk) // 8)
        if ty == 2:
            rows.setdefault((int(b_), int(j_)), {}).setdefault("tma", float(tt))
        if ty == 8:
            rows.setdefault((int(b_), int(j_)), {})["epi"] = float(tt)
    for ft, fb, fF in fin[:int(os.environ["TRACE_CHAIN"])]:
        print(f"  rollout {fb}: finalized at {ft:.1f} us, F={fF}")
        for j in range(k + 1):
            r_ = rows.get((fb, j))
            if not r_:
                continue
            c_ = r_.get("claim", (float("nan"), -1, -1))
            print(f"     row {j}: claim {c_[0]:6.1f} src {c_[1]} cl {c_[2]:2d}  tma {r_.get('tma', float('nan')):6.1f}  "
                  f"epi end {r_.get('epi', float('nan')):6.1f}")
