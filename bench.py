"""bench.py — throughput of the BubbleSpec hot path on B200 (BASELINE.json metric:
verified tokens/s/GPU at V=151936, k=8; mean accepted length; HBM GB/s).

One bench STEP = one RL step of the whole hot path on one synthetic
batch: pool put (a8) -> cross-rank exchange over NCCL (a9; a 1-rank communicator at N = 1,
so its cost is timed at every N) -> index build (a8) -> rollout begin -> first lookup (a1)
-> decoding until every rollout finished (EOS / max_len), each decoding step being the
synthetic target's rows (the model-forward stand-in) -> one bs_verify_commit_lookup launch:
verify (a2-a6), commit (a7) and the next step's lookup (a1).  Inputs (pools, prompt tails,
lengths, the 2.5 GB logit bank) are resident in HBM before the timed region; every rollout
reads its own logits rows (target mode "sample"), so rows are not shared through L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config q7]

Under torchrun (N > 1) every rank runs its own prompt shard (weak scaling), pools produced
on rank r are for rank (r+1)'s prompts and reach their owner through bs_draft_exchange
(NCCL over NVLink); timing is CUDA events, max over ranks.  Rank 0 prints one JSON line.
The default q7 run also measures the TINY and LC configurations (BASELINE.json configs[0],
configs[2]) and reports them under "other_configs"; warm-up RL step 0's emitted tokens are
compared with the oracle's on the CPU-baseline sample ("parity").
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]: "Qwen2.5-7B-shaped: V=151936, 256 rollouts, k=8, 4k-token
    # lognormal lengths, T=1.0, 1 GPU"
    "q7": dict(V=151936, prompts=16, G=16, k=8, M=32, T=1.0, top_p=1.0, mean_len=4096,
               sigma=0.6, cap=32768, nbank=131072, beta=15.75, match_rate=0.8, noise=0.02,
               G_pre=16, pool_frac=2.0 / 3.0),
    # configs[2]: "long-context: V=151936, 64 rollouts, 32k-token responses, k=16, draft pool
    # 8 drafts/prompt, top-p 0.95"
    "lc": dict(V=151936, prompts=8, G=8, k=16, M=32, T=1.0, top_p=0.95, mean_len=8192,
               sigma=0.6, cap=32768, nbank=131072, beta=15.75, match_rate=0.8, noise=0.02,
               G_pre=8, pool_frac=2.0 / 3.0),
    # configs[0]: the small case the oracle finishes in seconds
    "tiny": dict(V=1024, prompts=1, G=4, k=4, M=16, T=1.0, top_p=1.0, mean_len=64, sigma=0.0,
                 cap=64, nbank=256, beta=6.0, match_rate=0.9, noise=0.02, G_pre=4,
                 pool_frac=1.0, mode="position"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------- inputs
def make_step_inputs(cfg, step: int, rank: int, world: int):
    """Seeded synthetic inputs of one RL step for one rank (numpy, host)."""
    from workloads import TargetSpec, lognormal_lengths, make_pools, prompt_tails

    P, G, M = cfg["prompts"], cfg["G"], cfg["M"]
    spec = TargetSpec(V=cfg["V"], nbank=cfg["nbank"], mode=cfg.get("mode", "sample"), beta=cfg["beta"])
    base = step * 1_000_000
    # prompts owned by `rank` (prompt % world == rank): the rollouts of this rank
    own = np.array([base + i * world + rank for i in range(P)], dtype=np.int64)
    # pools this rank pre-generated in its bubble: for the prompts of rank+1
    prod_rank = (rank + 1) % world
    prod = np.array([base + i * world + prod_rank for i in range(P)], dtype=np.int64)
    tails_own = prompt_tails(7, own, M, cfg["V"])
    tails_prod = prompt_tails(7, prod, M, cfg["V"])
    n = P * G
    if cfg["sigma"] > 0:
        ml = lognormal_lengths(1000 * step + rank, n, cfg["mean_len"], cfg["sigma"], cfg["cap"])
    else:
        ml = np.full(n, cfg["mean_len"], np.int32)
    # pool sequence lengths: own lognormal draw, truncated at pool_frac * batch max (the
    # pre-generation halts when the slowest rank finishes; drafts ~0.63-0.72 x
    # response length)
    if cfg["sigma"] > 0:
        pl = lognormal_lengths(77 + 1000 * step + prod_rank, P * cfg["G_pre"], cfg["mean_len"],
                               cfg["sigma"], cfg["cap"])
    else:
        pl = np.full(P * cfg["G_pre"], cfg["mean_len"], np.int32)
    pl = np.minimum(pl, int(cfg["pool_frac"] * ml.max())).reshape(P, cfg["G_pre"])
    sp, off, tok = make_pools(spec, prod, tails_prod, cfg["G_pre"], pl, cfg["match_rate"],
                              noise=cfg["noise"], prefix=M)
    pid = np.repeat(own, G).astype(np.int32)
    trows = np.repeat(tails_own, G, axis=0).astype(np.int32)
    uids = ((np.uint64(step) << np.uint64(32)) + np.uint64(rank << 20)
            + np.arange(n, dtype=np.uint64))
    return dict(spec=spec, seq_prompt=sp.astype(np.int32), seq_off=off, tokens=tok, pid=pid,
                tails=trows, uids=uids, max_len=ml.astype(np.int32))


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        if os.environ.get("BS_NO_CLOCKS"):  # diagnostics only: no sampler
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("BS_CLOCK_MS", "200")], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append([time.time()] + parts)

    def window(self, t0, t1):
        """Keep only the samples taken inside [t0, t1] (host time): the sampler is started
        before the warm-up so its start-up does not overlap the timed region."""
        self.t0, self.t1 = t0, t1

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = getattr(self, "t0", -1e30), getattr(self, "t1", 1e30)
        rows = [r[1:] for r in self.rows if t0 <= r[0] <= t1] or [r[1:] for r in self.rows]
        self.rows = rows
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------------------- our arm


def nccl_comm(bs, dist, rank, world):
    """An NCCL communicator for bs_draft_exchange: the torch process group's ranks (N > 1),
    or a 1-rank communicator (N = 1) so the exchange runs, and is timed, at every N."""
    if world > 1:
        obj = [bs.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return bs.nccl_comm_init(obj[0], world, rank)
    return bs.nccl_comm_init(bs.nccl_unique_id(), 1, 0)


# ---------------------------------------------------------------------------- our arm
def run_ours(args, cfg, rank, world, dist, warmup, steps, bind_step0=False, e2e=True):
    import torch

    import paper_2605_08862_b200 as bs
    from paper_2605_08862_b200.engine import TARGET_MODES, RolloutEngine, Target

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    V, k = cfg["V"], cfg["k"]
    n = cfg["prompts"] * cfg["G"]
    total_steps = warmup + steps
    t0 = time.time()
    host = [make_step_inputs(cfg, s, rank, world) for s in range(total_steps)]
    log(f"[rank {rank}] inputs generated in {time.time() - t0:.1f}s")
    max_pool = max(len(h["tokens"]) for h in host) * max(1, world) + 16
    max_seqs = max(len(h["seq_prompt"]) for h in host) * max(1, world) + 4
    ctx = bs.Context(vocab=V, eos_id=-1, k_max=k, match_max=cfg["M"], max_rollouts=n,
                     pool_capacity_tokens=max_pool, pool_capacity_seqs=max_seqs,
                     device=dev.index, seed=0x5EED)
    spec = host[0]["spec"]
    bank = torch.empty((cfg["nbank"], V), dtype=torch.int16, device=dev)
    bs.bsx_synth_bank(bank, cfg["nbank"], V, spec.bank_seed, spec.beta, stream=stream)
    eng = RolloutEngine(ctx, n, k, cfg["T"], cfg["top_p"],
                        Target(bank, cfg["nbank"], spec.target_seed, TARGET_MODES[spec.mode]), stream=stream,
                        plain=cfg.get("plain", False), ngram=cfg.get("ngram"))
    if cfg.get("min_token_prob"):  # f4: confidence-scored suffix drafts (reading C1), from the first seal
        ctx.bs_draft_set_min_token_prob(cfg["min_token_prob"])
    comm = nccl_comm(bs, dist, rank, world)

    def dev_t(a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(dev)

    dins = [dict(sp=dev_t(h["seq_prompt"]), off=dev_t(h["seq_off"]), tok=dev_t(h["tokens"]),
                 ntok=int(len(h["tokens"])), pid=dev_t(h["pid"]), tails=dev_t(h["tails"]),
                 uids=dev_t(h["uids"].view(np.int64)), ml=dev_t(h["max_len"])) for h in host]
    torch.cuda.synchronize(dev)
    chunk = args.chunk
    graph = []

    def capture():
        """The decode graph: `chunk` steps of target rows -> bs_verify_commit_lookup, captured
        once (the lookup reads the sealed index through a device-resident descriptor, so the
        graph stays valid across RL steps; staleness is checked on the device)."""
        if not graph:
            graph.append(eng.capture(chunk))  # (runs one real, eager decoding step first)
        return graph[0]

    flags = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in range(2)]
    flag_ev = [torch.cuda.Event() for _ in range(2)]

    def replay_until_done(g, first=None):
        """Replay the decode graph until every rollout finished.  The all-finished flag of
        chunk c is copied to pinned memory and checked while chunk c+1 already runs, so the
        GPU does not idle on the host round trip (one extra, all-finished chunk at the end).
        first: an event pair around the first chunk (recorded outside the graph)."""
        steps_ = 0
        with torch.cuda.stream(stream):
            if first:
                first[0].record(stream)
            g.replay()
            if first:
                first[1].record(stream)
            steps_ += chunk
            c = 0
            while True:
                # live rollouts after chunk c (0: all finished), read while chunk c+1 runs
                flags[c % 2].copy_(eng.live_count(), non_blocking=True)
                flag_ev[c % 2].record(stream)
                g.replay()
                steps_ += chunk
                flag_ev[c % 2].synchronize()
                if int(flags[c % 2][0]) == 0:
                    break
                c += 1
        return steps_

    setup_parts = []

    def setup_step(s, d):
        with torch.cuda.stream(stream):
            t0 = time.perf_counter()
            ctx.bs_draft_pool_put(s, d["sp"], d["off"], d["tok"], d["ntok"], stream=stream)
            t1 = time.perf_counter()
            ctx.bs_draft_exchange(comm, rank, world, s, stream=stream)  # synchronises the stream
            t2 = time.perf_counter()
            eng.seal(s)  # synchronises the stream (index build is per RL step)
            t3 = time.perf_counter()
            eng.begin(d["uids"], d["pid"], d["tails"], d["ml"])
            setup_parts.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3))

    # per RL step, outside the graph: put, the exchange's three NCCL launches and its gather,
    # the seal's own kernels and CUB calls, begin, the first lookup
    D = cfg["M"] + k
    launches_rl = 1 + 4 + (4 + 9 * D) + 2

    setup_ms = []

    def rl_step(s, rec, evs=None):
        t_set = time.perf_counter()
        setup_step(s + 1, dins[s])  # (the seal synchronises: host time covers the device work)
        setup_ms.append((time.perf_counter() - t_set) * 1e3)
        g = capture()
        if evs:
            evs[0].record(stream)
        steps_ = replay_until_done(g, evs[2:] if evs else None)
        if evs:
            evs[1].record(stream)
        rec["launches"] += launches_rl
        rec["decode_steps"] += steps_
        rec["launches"] += steps_ * eng.launches_per_step
        rec["launches"] += steps_ // chunk - 1  # bs_rollout_live per checked chunk (the done flag)
        return steps_

    rec0 = dict(launches=0, decode_steps=0)
    # nvidia-smi is started before the warm-up (its start-up stays outside the timed region);
    # only its samples inside the timed window are kept
    clocks = ClockSampler(dev.index)
    clocks.start()
    # ---- warm-up (RL step 0's responses are kept for the oracle comparison)
    resp0 = None
    for s in range(warmup):
        if s == 0 and bind_step0:
            Lmax = int(host[0]["max_len"].max())
            resp = torch.full((n, Lmax), -1, dtype=torch.int32, device=dev)
            ctx.bs_rollout_bind_output(resp, Lmax)
            rl_step(s, dict(rec0))
            torch.cuda.synchronize(dev)
            ctx.bs_rollout_bind_output(None)
            resp0 = resp.cpu().numpy()
            del resp
        else:
            rl_step(s, dict(rec0))
    torch.cuda.synchronize(dev)
    if ctx.bs_sync_status():
        raise SystemExit("device error word set during warm-up")
    # ---- steady state (untimed): the first chunk of a fresh RL step, full live batch; the
    # chunk replay is bracketed by two events outside the graph
    ctx.bs_stats_read(reset=True, stream=stream)
    setup_step(10_000, dins[total_steps - 1])
    e_s0, e_s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e_s0.record(stream)
        capture().replay()
        e_s1.record(stream)
    torch.cuda.synchronize(dev)
    steady_ms = e_s0.elapsed_time(e_s1)
    sst = eng.stats(reset=True)
    with torch.cuda.stream(stream):
        while not eng.all_finished():  # finish that RL step (untimed)
            capture().replay()
    torch.cuda.synchronize(dev)
    ctx.bs_stats_read(reset=True, stream=stream)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # ---- timed region
    rec = dict(rec0)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_host0 = time.time()
    start.record(stream)
    for i, s in enumerate(range(warmup, total_steps)):
        rl_step(s, rec, evs[i])
    end.record(stream)
    torch.cuda.synchronize(dev)
    log("[timed] decode ms per RL step: " + " ".join(f"{e[0].elapsed_time(e[1]):.1f}" for e in evs))
    log("[timed] setup (put, exchange, seal, begin) host ms per RL step: "
        + " ".join(f"{x:.1f}" for x in setup_ms[-len(evs):]) + "  (put / exchange / seal: "
        + " ".join(f"{a_:.1f}/{b_:.1f}/{c_:.1f}" for a_, b_, c_ in setup_parts[-len(evs):]) + ")")
    t_host1 = time.time()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.window(t_host0, t_host1)
    clk = clocks.stop()
    elapsed_ms = start.elapsed_time(end)
    decode_ms = sum(e[0].elapsed_time(e[1]) for e in evs)
    first_ms = sum(e[2].elapsed_time(e[3]) for e in evs)
    st = eng.stats(reset=True)
    word = ctx.bs_sync_status()
    if word:
        raise SystemExit(f"device error word 0x{word:x} in the timed region: no number is reported")
    # ---- e2e: the same RL steps through the public API from pinned HOST buffers
    e2e_r = run_e2e(args, cfg, ctx, eng, host[warmup:], stream, dev, capture, comm, rank, world, dist,
                    replay_until_done, setup_step) if e2e else None
    if e2e_r is not None and ctx.bs_sync_status():
        raise SystemExit("device error word set in the e2e leg")
    info = ctx.bsx_launch_info()
    # ---- gather over ranks
    vals = torch.tensor([elapsed_ms, float(st["tokens"]), e2e_r["ms"] if e2e_r else 0.0,
                         float(e2e_r["tokens"]) if e2e_r else 0.0, decode_ms, float(st["rows_needed"]),
                         float(st["rows_verified"])], dtype=torch.float64, device=dev)
    if dist is not None:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        agg = dict(elapsed_ms=float(mx[0]), tokens=float(sm[1]), e2e_ms=float(mx[2]), e2e_tokens=float(sm[3]),
                   decode_ms=float(mx[4]), rows_needed=float(sm[5]), rows_verified=float(sm[6]))
    else:
        agg = dict(elapsed_ms=elapsed_ms, tokens=float(st["tokens"]), e2e_ms=e2e_r["ms"] if e2e_r else 0.0,
                   e2e_tokens=float(e2e_r["tokens"]) if e2e_r else 0.0, decode_ms=decode_ms,
                   rows_needed=float(st["rows_needed"]), rows_verified=float(st["rows_verified"]))
    bs.nccl_comm_destroy(comm)
    return dict(agg=agg, st=st, rec=rec, clocks=clk, steady_ms=steady_ms, sst=sst, e2e=e2e_r,
                first_ms=first_ms, decode_ms_local=decode_ms, resp0=resp0, info=info, n=n)


def run_e2e(args, cfg, ctx, eng, host, stream, dev, capture, comm, rank, world, dist, replay_until_done,
            setup_step):
    """End-to-end through the public API: every RL step copies its inputs host->device from
    pinned memory (pools, prompt tails, uids, lengths) and reads the generated responses
    back device->host, inside the timed region."""
    import torch

    n = cfg["prompts"] * cfg["G"]
    Lmax = max(int(h["max_len"].max()) for h in host)
    resp = torch.full((n, Lmax), -1, dtype=torch.int32, device=dev)
    ctx.bs_rollout_bind_output(resp, Lmax)
    pinned = []
    for h in host:
        pinned.append({key: torch.from_numpy(np.ascontiguousarray(h[key] if key != "uids" else
                                                                  h[key].view(np.int64))).pin_memory()
                       for key in ("seq_prompt", "seq_off", "tokens", "pid", "tails", "uids",
                                   "max_len")})
    resp_host = torch.empty((n, Lmax), dtype=torch.int32).pin_memory()
    h2d = sum(int(t.numel() * t.element_size()) for t in pinned[0].values())
    d2h = int(resp_host.numel() * resp_host.element_size())
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    ctx.bs_stats_read(reset=True, stream=stream)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in pinned]
    for i, p in enumerate(pinned):
        with torch.cuda.stream(stream):
            d = {key: t.to(dev, non_blocking=True) for key, t in p.items()}
        setup_step(20_000 + i, dict(sp=d["seq_prompt"], off=d["seq_off"], tok=d["tokens"],
                                     ntok=int(p["tokens"].numel()), pid=d["pid"], tails=d["tails"],
                                     uids=d["uids"], ml=d["max_len"]))
        evs[i][0].record(stream)
        replay_until_done(capture())
        evs[i][1].record(stream)
        with torch.cuda.stream(stream):
            resp_host.copy_(resp, non_blocking=True)
    end.record(stream)
    torch.cuda.synchronize(dev)
    ms = start.elapsed_time(end)
    log("[e2e] decode ms per RL step: " + " ".join(f"{e[0].elapsed_time(e[1]):.1f}" for e in evs) +
        f"; total {ms:.1f}")
    st = eng.stats(reset=True)
    ctx.bs_rollout_bind_output(None)
    return dict(ms=ms, tokens=st["tokens"], h2d=h2d, d2h=d2h)


# ---------------------------------------------------------------------------- CPU oracle
_ORC = {}


def _oracle_worker(arg):
    """One host core: whole decoding steps of its rollouts, round-robin, until its share of
    the time budget of ORACLE time (draft lookup + Alg. 1 step; row generation excluded)."""
    from oracle.rollout import OracleRollout, bank_row_fn, pools_by_prompt, step

    which, budget = arg
    j = _ORC
    h, cfg = j["h"], j["cfg"]
    pools = pools_by_prompt(h["seq_prompt"], h["seq_off"], h["tokens"])
    fn = bank_row_fn(h["spec"])
    ros = {b: OracleRollout(prompt=int(h["pid"][b]), uid=int(h["uids"][b]),
                            context=[int(x) for x in h["tails"][b]], max_len=int(h["max_len"][b]))
           for b in which}
    timers = {}
    tokens = nsteps = 0
    i = 0
    while timers.get("oracle_s", 0.0) < budget and any(not r.finished for r in ros.values()):
        ro = ros[which[i % len(which)]]
        if not ro.finished:
            out = step(ro, pools, fn, k=cfg["k"], M=cfg["M"], Lmin=1, T=cfg["T"], top_p=cfg["top_p"],
                       seed=0x5EED, eos=-1, timers=timers)
            if out is not None:
                tokens += len(out.tokens)
                nsteps += 1
        i += 1
    return dict(tokens=tokens, steps=nsteps, rows=timers.get("rows", 0), secs=timers.get("oracle_s", 0.0),
                gen={b: r.generated for b, r in ros.items()})


def cpu_oracle_sample(cfg, budget_s: float, cores: int, rank: int = 0, world: int = 1):
    """The oracle as it stands, on `cores` host cores (independent rollouts in forked
    processes, each plain and single-threaded), on a bounded sample of RL step 0 of the same
    workload.  Returns (tokens/s, sample description, generated tokens per rollout)."""
    import multiprocessing as mp

    h = make_step_inputs(cfg, 0, rank, world)
    _ORC.clear()
    _ORC.update(h=h, cfg=cfg)
    n = len(h["pid"])
    order = np.argsort(h["pid"], kind="stable")
    groups = [list(map(int, g)) for g in np.array_split(order, cores) if len(g)]
    if cores == 1:
        res = [_oracle_worker((groups[0], budget_s))]
    else:
        with mp.get_context("fork").Pool(len(groups)) as pool:
            res = pool.map(_oracle_worker, [(g, budget_s) for g in groups], chunksize=1)
    tokens = sum(r["tokens"] for r in res)
    secs = max(r["secs"] for r in res)  # the processes run concurrently
    gen = {}
    for r in res:
        gen.update(r["gen"])
    desc = (f"{sum(r['steps'] for r in res)} decoding steps (lookup + Alg. 1 step) of the {n} rollouts of "
            f"RL step 0 on {len(groups)} core(s), {sum(r['rows'] for r in res)} logits rows, {tokens} tokens; "
            f"oracle time only (the slowest core's)")
    return tokens / secs, desc, gen


def host_cpu():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


def parity_check(resp0, gen):
    """Warm-up RL step 0's emitted tokens (GPU) vs the oracle's on the sampled steps."""
    if resp0 is None:
        return None
    bad, toks = 0, 0
    for b, g in gen.items():
        toks += len(g)
        if [int(x) for x in resp0[b, : len(g)]] != list(g):
            bad += 1
    return {"rollouts": len(gen), "tokens": toks, "mismatched_rollouts": bad,
            "what": "warm-up RL step 0, every rollout's tokens from the oracle sample's decoding steps"}


def summarize(cfg, name, r, args, peaks_hbm):
    """Numbers of one configuration from run_ours' result."""
    agg, st = r["agg"], r["st"]
    V = cfg["V"]
    row_bytes = 2 * V
    value = agg["tokens"] / (agg["elapsed_ms"] / 1e3)
    achieved = agg["rows_needed"] * row_bytes / (agg["decode_ms"] * 1e-3) / 1e9
    moved = agg["rows_verified"] * row_bytes / (agg["decode_ms"] * 1e-3) / 1e9
    steady = r["sst"]["rows_needed"] * row_bytes / (r["steady_ms"] * 1e-3) / 1e9
    steady_moved = r["sst"]["rows_verified"] * row_bytes / (r["steady_ms"] * 1e-3) / 1e9
    return dict(value=value, ms_per_step=agg["elapsed_ms"] / args_steps(args, name),
                achieved=achieved, moved=moved, steady=steady, steady_moved=steady_moved,
                frac=achieved / peaks_hbm, steady_frac=steady / peaks_hbm,
                decode_ms=agg["decode_ms"], elapsed_ms=agg["elapsed_ms"])


def args_steps(args, name):
    return args.steps if name == args.config else EXTRA_STEPS[1]


EXTRA_STEPS = (3, 2)  # (warm-up, timed) RL steps of the extra TINY / LC lines
SWEEP_STEPS = (1, 1)  # (warm-up, timed) RL steps of each acceptance-sweep point


def sweep_configs():
    """BASELINE.json configs[4] ("acceptance sweep: draft match rate 0-90%, k in {2,4,8,16} ...
    vs plain decoding"), at one GPU on a shortened Q7 workload (mean length 1024): k in
    {2, 4, 8, 16} at match rate 0.8, match rate in {0, 0.5, 0.95} at k = 8, and plain decoding
    (no drafts: one sample per decoding step)."""
    base = dict(CONFIGS["q7"], mean_len=1024, cap=8192)
    pts = [("k%d_r0.8" % k, dict(base, k=k)) for k in (2, 4, 8, 16)]
    pts += [("k8_r%g" % r, dict(base, match_rate=r)) for r in (0.0, 0.5, 0.95)]
    pts.append(("plain", dict(base, k=8, plain=True)))
    # f4 draft-source ablation (the paper's Table 7): the n-gram linear-scan drafter
    # on the same workload as k8_r0.8 (suffix index)
    pts.append(("ngram_k8_r0.8", dict(base, ngram=(1, 32))))
    # ... and confidence-scored suffix drafts (reading C1, Arctic-style min_token_prob)
    pts += [("conf%g_k8_r0.8" % t, dict(base, min_token_prob=t)) for t in (0.3, 0.6)]
    return pts


def workload_str(name, cfg):
    return (f"{name}: V={cfg['V']}, {cfg['prompts'] * cfg['G']} rollouts/GPU ({cfg['prompts']} prompts x "
            f"{cfg['G']}), k={cfg['k']}, lognormal lengths mean {cfg['mean_len']} sigma {cfg['sigma']} cap "
            f"{cfg['cap']}, T={cfg['T']}, top_p={cfg['top_p']}, pools {cfg['G_pre']}/prompt, match rate "
            f"{cfg['match_rate']}, target rows per rollout (mode sample)")


# ---------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="q7")
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the TINY / LC lines")
    ap.add_argument("--no-sweep", action="store_true", help="skip the acceptance sweep (configs[4])")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        log(f"note: WORLD_SIZE={world}, --gpus={args.gpus}")
    metric = "verified tokens/sec/GPU at V=151936, k=8; mean accepted length; HBM GB/s"
    unit = "verified tokens/s"
    workload = workload_str(args.config, cfg)
    ncores, cpu_model = host_cpu()

    if args.impl == "reference":
        if rank != 0:
            return
        vals = []
        desc = ""
        for _ in range(args.steps):  # each step: a bounded sample on every host core
            v, desc, _gen = cpu_oracle_sample(cfg, args.cpu_budget / max(1, args.steps), ncores)
            vals.append(v)
        val = float(np.median(vals))
        out = {"impl": "reference", "metric": metric, "value": val, "unit": unit,
               "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "u64", "data": "synthetic",
               "config": {"workload": workload},
               "cpu_baseline": {"value": val, "unit": unit, "cores": ncores, "cpu": cpu_model,
                                "kind": "oracle", "sample": desc},
               "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl")
        dist = tdist
    r = run_ours(args, cfg, rank, world, dist, args.warmup, args.steps, bind_step0=(rank == 0))
    extra = {}
    if args.config == "q7" and not args.no_extra:
        for name in ("tiny", "lc"):
            extra[name] = (CONFIGS[name], run_ours(args, CONFIGS[name], rank, world, dist, *EXTRA_STEPS,
                                                   e2e=False))
    f_rows = {}
    if args.config == "q7" and not args.no_extra and rank == 0:
        # the NEXT rows of SURVEY §8(f) on this GPU: f2 unified attention (the paper's Table 2
        # setting) and f1 bubble pre-generation (virtual DP ranks); scripts/ hold the drivers
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import attn_bench
        import bubble_pregen
        import lmhead_bench

        f_rows["unified_attention"] = attn_bench.main(["--iters", "10"], quiet=True)
        f_rows["lm_head_fused_stats"] = lmhead_bench.main(["--rows", "256,2304", "--iters", "5"], quiet=True)
        summ, rep = bubble_pregen.main(["--steps", "3"], quiet=True)
        f_rows["bubble_pregen"] = dict(summ, steps=[{k2: v for k2, v in r_.items() if k2 in (
            "rl_step", "step_ms", "bubble_frac", "acceptance_length", "mean_decode_steps_per_rollout",
            "slowest_rank_decode_steps", "pregen_tokens")} for r_ in rep])
    sweep = []
    if args.config == "q7" and not args.no_sweep and not args.no_extra:
        for name, c in sweep_configs():
            sweep.append((name, c, run_ours(args, c, rank, world, dist, *SWEEP_STEPS, e2e=False)))
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    st, rec = r["st"], r["rec"]
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if hbm else "fallback 6650 GB/s"
    hbm = hbm or 6650.0
    sm = summarize(cfg, args.config, r, args, hbm)
    cpu, parity = None, None
    if not args.no_cpu_baseline:
        cv, desc, gen = cpu_oracle_sample(cfg, args.cpu_budget, ncores)
        cv1, desc1, _ = cpu_oracle_sample(cfg, args.cpu_budget / 2, 1)
        cpu = {"value": cv, "unit": unit, "cores": ncores, "cpu": cpu_model, "kind": "oracle", "sample": desc,
               "single_core": {"value": cv1, "sample": desc1}}
        parity = parity_check(r["resp0"], gen)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "verify_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except ValueError:
            traffic = None
    others = {}
    for name, (c2, r2) in extra.items():
        s2 = summarize(c2, name, r2, args, hbm)
        others[name] = {"workload": workload_str(name, c2), "value": s2["value"], "unit": unit,
                        "ms_per_step": s2["ms_per_step"], "steps": EXTRA_STEPS[1], "warmup": EXTRA_STEPS[0],
                        "acceptance_length": r2["st"]["acceptance_length"],
                        "draft_length": r2["st"]["draft_length"], "tokens": int(r2["agg"]["tokens"]),
                        "roofline_frac": s2["frac"], "steady_frac": s2["steady_frac"],
                        "hbm_gbs": {"algorithmic": s2["achieved"], "steady_algorithmic": s2["steady"]}}
    sweep_out = []
    plain_steps = None
    for name, c2, r2 in sweep:
        s2 = summarize(c2, name, r2, args, hbm)
        s2["ms_per_step"] = r2["agg"]["elapsed_ms"] / SWEEP_STEPS[1]
        rec2 = {"point": name, "k": c2["k"], "match_rate": c2["match_rate"], "plain": c2.get("plain", False),
                "drafter": "none" if c2.get("plain") else ("ngram" if c2.get("ngram") else (
                    "suffix index, min_token_prob %g" % c2["min_token_prob"] if c2.get("min_token_prob")
                    else "suffix index")),
                "value": s2["value"], "unit": unit, "ms_per_rl_step": s2["ms_per_step"],
                "acceptance_length": r2["st"]["acceptance_length"],
                "decode_steps_per_rollout": r2["st"]["decode_steps"] / r2["n"],
                "roofline_frac": s2["frac"], "steady_frac": s2["steady_frac"]}
        if c2.get("plain"):
            plain_steps = rec2["decode_steps_per_rollout"]
        sweep_out.append(rec2)
    for rec2 in sweep_out:
        if plain_steps:
            rec2["decode_step_reduction_vs_plain"] = 1 - rec2["decode_steps_per_rollout"] / plain_steps
    out = {
        "metric": metric, "value": sm["value"], "unit": unit, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sm["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded counter-hash bank of 8192 bf16 logit rows, perturbed pools)",
        "config": {"workload": workload, "parallelism": f"dp{args.gpus}",
                   "rollouts": cfg["prompts"] * cfg["G"] * args.gpus,
                   "l2": "inputs larger than L2 (2.5 GB logit bank; every rollout reads its own rows)",
                   "graph_chunk": args.chunk, "verify_launch": r["info"]},
        "per_gpu_value": sm["value"] / args.gpus,
        "acceptance_length": st["acceptance_length"], "draft_length": st["draft_length"],
        "acceptance_rate": st["acceptance_rate"], "decode_steps": st["decode_steps"],
        "tokens": int(r["agg"]["tokens"]),
        "hbm_gbs": {"algorithmic": sm["achieved"], "moved": sm["moved"],
                    "steady_algorithmic": sm["steady"], "steady_moved": sm["steady_moved"]},
        "roofline": {"bound": "hbm", "achieved": sm["achieved"], "peak": hbm, "unit": "GB/s",
                     "frac": sm["achieved"] / hbm, "traffic": traffic,
                     "kernel": "decoding step = bs_verify_commit_lookup (verify_cluster_kernel: plan, rows, "
                               "fused commit and next-draft lookup) + the synthetic model's row kernel; "
                               "timed by CUDA events around the decode-graph replays of the timed RL steps "
                               "(outside the graphs), algorithmic bytes = rows Alg. 1 needs x 2V",
                     "decode_ms": sm["decode_ms"], "timed_ms": sm["elapsed_ms"],
                     "peak_source": peak_src, "steady_frac": sm["steady_frac"],
                     "steady_what": "first 64-step chunk of a fresh RL step (all rollouts live), events "
                                    "around that one graph replay"},
        "clocks": r["clocks"],
        "e2e": {"value": r["agg"]["e2e_tokens"] / (r["agg"]["e2e_ms"] / 1e3), "unit": unit,
                "h2d_bytes_per_step": r["e2e"]["h2d"], "d2h_bytes_per_step": r["e2e"]["d2h"]},
        "gpu_launches": rec["launches"],
        "cpu_baseline": cpu,
        "parity": parity,
        "other_configs": others,
        "next_rows": f_rows or None,
        "sweep": {"workload": "BASELINE.json configs[4] at 1 GPU: q7 shape with mean length 1024 (cap 8192), "
                              "1 warm-up + 1 timed RL step per point; plain = no drafts",
                  "points": sweep_out} if sweep_out else None,
    }
    print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
