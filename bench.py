"""bench.py — throughput of the BubbleSpec hot path on B200 (BASELINE.json metric:
verified tokens/s/GPU at V=151936, k=8; mean accepted length; HBM GB/s).

One bench STEP = one RL step of the whole hot path on one synthetic
batch: pool put (a8) -> cross-rank exchange (a9, N > 1) -> index build (a8) -> rollout begin
-> first lookup (a1) -> decoding until every rollout finished (EOS / max_len), each decoding
step being synthetic target rows -> one bs_verify_commit_lookup launch: verify (a2-a6),
commit (a7) and the next step's lookup (a1).  Inputs (pools, prompt
tails, lengths, the 2.5 GB logit bank) are resident in HBM before the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config q7]

Under torchrun (N > 1) every rank runs its own prompt shard (weak scaling), pools produced
on rank r are for rank (r+1)'s prompts and reach their owner through bs_draft_exchange
(NCCL over NVLink); timing is CUDA events, max over ranks.  Rank 0 prints one JSON line.
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
               sigma=0.6, cap=32768, nbank=8192, beta=15.75, match_rate=0.8, noise=0.02,
               G_pre=16, pool_frac=2.0 / 3.0),
    # configs[2]: "long-context: V=151936, 64 rollouts, 32k-token responses, k=16, draft pool
    # 8 drafts/prompt, top-p 0.95"
    "lc": dict(V=151936, prompts=8, G=8, k=16, M=32, T=1.0, top_p=0.95, mean_len=8192,
               sigma=0.6, cap=32768, nbank=8192, beta=15.75, match_rate=0.8, noise=0.02,
               G_pre=8, pool_frac=2.0 / 3.0),
    # configs[0]: the small case the oracle finishes in seconds
    "tiny": dict(V=1024, prompts=1, G=4, k=4, M=16, T=1.0, top_p=1.0, mean_len=64, sigma=0.0,
                 cap=64, nbank=256, beta=6.0, match_rate=0.9, noise=0.02, G_pre=4,
                 pool_frac=1.0),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------- inputs
def make_step_inputs(cfg, step: int, rank: int, world: int):
    """Seeded synthetic inputs of one RL step for one rank (numpy, host)."""
    from workloads import TargetSpec, lognormal_lengths, make_pools, prompt_tails

    P, G, M = cfg["prompts"], cfg["G"], cfg["M"]
    spec = TargetSpec(V=cfg["V"], nbank=cfg["nbank"], mode="position", beta=cfg["beta"])
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
def run_ours(args, cfg, rank, world, dist):
    import torch

    import paper_2605_08862_b200 as bs
    from paper_2605_08862_b200.engine import RolloutEngine, Target

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    V, k = cfg["V"], cfg["k"]
    n = cfg["prompts"] * cfg["G"]
    total_steps = args.warmup + args.steps
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
                        Target(bank, cfg["nbank"], spec.target_seed, 0), stream=stream)
    comm = None
    if world > 1:
        uid = bs.nccl_unique_id() if rank == 0 else None
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        comm = bs.nccl_comm_init(obj[0], world, rank)

    def dev_t(a, dtype=None):
        t = torch.from_numpy(np.ascontiguousarray(a))
        return t.to(dev, non_blocking=False) if dtype is None else t.to(dtype).to(dev)

    dins = [dict(sp=dev_t(h["seq_prompt"]), off=dev_t(h["seq_off"]), tok=dev_t(h["tokens"]),
                 ntok=int(len(h["tokens"])), pid=dev_t(h["pid"]), tails=dev_t(h["tails"]),
                 uids=dev_t(h["uids"].view(np.int64)), ml=dev_t(h["max_len"])) for h in host]
    torch.cuda.synchronize(dev)
    chunk = args.chunk
    # verify-op timing events captured inside the graph (external event-record nodes)
    ev_s = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(chunk)]
    ev_e = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(chunk)]

    graphs = {}

    def capture(instrument=False):
        """The decode graph (captured once: the library reads the sealed index through a
        device-resident descriptor, so the graph stays valid across RL steps)."""
        if instrument not in graphs:
            graphs[instrument] = capture_new(instrument)
        return graphs[instrument]

    def capture_new(instrument=False):
        """One graph of `chunk` decode iterations.  Event-record nodes cost several us each
        inside a graph, so the timed graph has none; the instrumented twin (events around
        every bs_verify_step) is replayed separately on the same deterministic work."""
        with torch.cuda.stream(stream):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for i in range(chunk):
                    c, t = ctx, eng.target
                    # the drafts of this step: from the previous verify launch (fused lookup;
                    # the first step's from eng.begin)
                    c.bsx_target_rows(eng.slots, eng.draft, eng.draft_len, k, t.target_seed,
                                      t.mode, t.nbank, eng.row_index, stream=stream)
                    if instrument:
                        ev_s[i].record(stream)
                    c.bs_verify_commit_lookup(eng.rl_step, eng.slots, t.bank, eng.row_index, V, eng.draft,
                                              eng.draft_len, k, eng.T, eng.top_p, eng.out_tokens,
                                              eng.out_len, eng.out_acc, eng.finished, eng.match_len,
                                              stream=stream)
                    if instrument:
                        ev_e[i].record(stream)
        return g

    phases = os.environ.get("BS_BENCH_PHASES")  # diagnostics: host wall per RL-step phase
    flags = [torch.zeros(1, dtype=torch.bool).pin_memory() for _ in range(2)]
    flag_ev = [torch.cuda.Event() for _ in range(2)]

    def replay_until_done(g):
        """Replay the decode graph until every rollout finished.  The all-finished flag of
        chunk c is copied to pinned memory and checked while chunk c+1 already runs, so the
        GPU does not idle on the host round trip (one extra, all-finished chunk at the end)."""
        steps = 0
        with torch.cuda.stream(stream):
            g.replay()
            steps += chunk
            c = 0
            while True:
                flags[c % 2].copy_(eng.finished.all().view(1), non_blocking=True)
                flag_ev[c % 2].record(stream)
                g.replay()
                steps += chunk
                flag_ev[c % 2].synchronize()
                if bool(flags[c % 2][0]):
                    break
                c += 1
        return steps

    def rl_step(s, rec, instrument=False):
        d = dins[s]
        tp = [time.perf_counter()]

        def mark():
            if phases:
                stream.synchronize()
                tp.append(time.perf_counter())
        with torch.cuda.stream(stream):
            ctx.bs_draft_pool_put(s + 1, d["sp"], d["off"], d["tok"], d["ntok"], stream=stream)
            mark()
            if comm is not None:
                ctx.bs_draft_exchange(comm, rank, world, s + 1, stream=stream)
            eng.seal(s + 1)  # synchronises the stream (index build is per RL step)
            mark()
            eng.begin(d["uids"], d["pid"], d["tails"], d["ml"])
            mark()
        g = capture(instrument)
        mark()
        rec["launches"] += 2 + int(eng.fuse_lookup) + rec["seal_launches"]  # put, begin, first lookup
        steps, chunks = 0, 0
        if instrument:  # events are re-recorded by every replay: one chunk at a time
            while True:
                with torch.cuda.stream(stream):
                    g.replay()
                    done = bool(eng.finished.all().item())  # one host sync per chunk
                steps += chunk
                vt = sum(ev_s[i].elapsed_time(ev_e[i]) for i in range(chunk))
                rec["verify_ms"] += vt
                if chunks == 0:
                    rec["verify_ms_steady"] += vt
                    rec["steady_steps"] += chunk
                chunks += 1
                if done:
                    break
        else:  # the finished check of chunk c overlaps the replay of chunk c+1
            steps += replay_until_done(g)
        mark()
        rec["decode_steps"] += steps
        rec["launches"] += steps * eng.launches_per_step
        if phases:
            dt = [1e3 * (b - a) for a, b in zip(tp, tp[1:])]
            log("[phases ms] put %.1f seal %.1f begin %.1f capture %.1f decode %.1f" % tuple(dt[:5]))
        return steps

    # seal launch count: our own kernels + CUB device calls per level
    D = cfg["M"] + k
    rec0 = dict(launches=0, verify_ms=0.0, verify_ms_steady=0.0, steady_steps=0, decode_steps=0,
                seal_launches=4 + 9 * D)
    # nvidia-smi is started before the warm-up (its start-up stays outside the timed region);
    # only its samples inside the timed window are kept
    clocks = ClockSampler(dev.index)
    clocks.start()
    # ---- warmup
    for s in range(args.warmup):
        rl_step(s, dict(rec0))
    ctx.bs_stats_read(reset=True, stream=stream)
    # steady-state row counters need the first chunk separately: read stats after chunk 0
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    # ---- (untimed, before the timed region: it also settles the device) the verify op's
    # device time on the same work: instrumented replay of the RL steps that are timed next
    # (deterministic: same pools, uids and Philox stream -> identical rows)
    reci = dict(rec0)
    for s in range(args.warmup, total_steps):
        rl_step(s, reci, instrument=True)
    torch.cuda.synchronize(dev)
    sti = eng.stats(reset=True)
    # ---- steady-state kernel phase: full live batch, first chunk of a fresh RL step
    s_last = total_steps - 1
    d = dins[s_last]
    with torch.cuda.stream(stream):
        ctx.bs_draft_pool_put(10_000, d["sp"], d["off"], d["tok"], d["ntok"], stream=stream)
        if comm is not None:
            ctx.bs_draft_exchange(comm, rank, world, 10_000, stream=stream)
        eng.seal(10_000)
        eng.begin(d["uids"], d["pid"], d["tails"], d["ml"])
    g = capture(instrument=True)
    with torch.cuda.stream(stream):
        g.replay()
    torch.cuda.synchronize(dev)
    steady_ms = sum(ev_s[i].elapsed_time(ev_e[i]) for i in range(chunk))
    sst = eng.stats(reset=True)
    rec = dict(rec0)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_host0 = time.time()
    start.record(stream)
    for s in range(args.warmup, total_steps):
        rl_step(s, rec)
    end.record(stream)
    torch.cuda.synchronize(dev)
    t_host1 = time.time()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.window(t_host0, t_host1)
    clk = clocks.stop()
    elapsed_ms = start.elapsed_time(end)
    st = eng.stats(reset=True)
    if sti["tokens"] != st["tokens"] or sti["rows_verified"] != st["rows_verified"]:
        log(f"note: instrumented replay differs ({sti['tokens']} vs {st['tokens']} tokens, "
            f"{sti['rows_verified']} vs {st['rows_verified']} rows)")
    rec["verify_ms"] = reci["verify_ms"]
    rec["verify_rows_verified"] = sti["rows_verified"]
    rec["verify_rows_needed"] = sti["rows_needed"]
    # ---- e2e: the same RL steps through the public API from pinned HOST buffers
    e2e = run_e2e(args, cfg, ctx, eng, host, stream, dev, capture, comm, rank, world, dist, replay_until_done)
    # ---- gather over ranks
    import torch as _t

    vals = _t.tensor([elapsed_ms, float(st["tokens"]), e2e["ms"], float(e2e["tokens"])],
                     dtype=_t.float64, device=dev)
    if dist is not None:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        elapsed_all, tokens_all = float(mx[0]), float(sm[1])
        e2e_ms_all, e2e_tok_all = float(mx[2]), float(sm[3])
    else:
        elapsed_all, tokens_all = elapsed_ms, float(st["tokens"])
        e2e_ms_all, e2e_tok_all = e2e["ms"], float(e2e["tokens"])
    if comm is not None:
        bs.nccl_comm_destroy(comm)
    return dict(elapsed_ms=elapsed_all, tokens=tokens_all, st=st, rec=rec, clocks=clk,
                steady_ms=steady_ms, sst=sst, e2e=e2e, e2e_ms=e2e_ms_all, e2e_tokens=e2e_tok_all)


def run_e2e(args, cfg, ctx, eng, host, stream, dev, capture, comm, rank, world, dist, replay_until_done):
    """End-to-end through the public API: every RL step copies its inputs host->device from
    pinned memory (pools, prompt tails, uids, lengths) and reads the generated responses
    back device->host, inside the timed region."""
    import torch

    n = cfg["prompts"] * cfg["G"]
    Lmax = max(int(h["max_len"].max()) for h in host)
    resp = torch.full((n, Lmax), -1, dtype=torch.int32, device=dev)
    ctx.bs_rollout_bind_output(resp, Lmax)
    pinned = []
    for h in host[args.warmup:]:
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
    for i, p in enumerate(pinned):
        s = 20_000 + i
        with torch.cuda.stream(stream):
            d = {key: t.to(dev, non_blocking=True) for key, t in p.items()}
            ctx.bs_draft_pool_put(s, d["seq_prompt"], d["seq_off"], d["tokens"],
                                  int(p["tokens"].numel()), stream=stream)
            if comm is not None:
                ctx.bs_draft_exchange(comm, rank, world, s, stream=stream)
            eng.seal(s)
            eng.begin(d["uids"], d["pid"], d["tails"], d["max_len"])
        g = capture()
        replay_until_done(g)
        with torch.cuda.stream(stream):
            resp_host.copy_(resp, non_blocking=True)
    end.record(stream)
    torch.cuda.synchronize(dev)
    ms = start.elapsed_time(end)
    st = eng.stats(reset=True)
    ctx.bs_rollout_bind_output(None)
    return dict(ms=ms, tokens=st["tokens"], h2d=h2d, d2h=d2h)


# ---------------------------------------------------------------------------- CPU oracle
def cpu_oracle_sample(cfg, budget_s: float, rank: int = 0, world: int = 1):
    """The oracle as it stands on the host cores, on a bounded sample of the same workload:
    whole decoding steps of the first rollouts of one RL step until ~budget_s of oracle
    time.  Returns (tokens/s, sample description, oracle seconds)."""
    import oracle
    from oracle.rollout import OracleRollout, bank_row_fn, pools_by_prompt, step

    h = make_step_inputs(cfg, 0, rank, world)
    # the single-GPU workload: pools of the rank's own prompts (world == 1 -> identical)
    pools = pools_by_prompt(h["seq_prompt"], h["seq_off"], h["tokens"])
    fn = bank_row_fn(h["spec"])
    ros = [OracleRollout(prompt=int(h["pid"][b]), uid=int(h["uids"][b]),
                         context=[int(x) for x in h["tails"][b]], max_len=int(h["max_len"][b]))
           for b in range(len(h["pid"]))]
    timers = {}
    tokens, nsteps = 0, 0
    b = 0
    while timers.get("oracle_s", 0.0) < budget_s:
        ro = ros[b % len(ros)]
        if not ro.finished:
            out = step(ro, pools, fn, k=cfg["k"], M=cfg["M"], Lmin=1, T=cfg["T"],
                       top_p=cfg["top_p"], seed=0x5EED, eos=-1, timers=timers)
            if out is not None:
                tokens += len(out.tokens)
                nsteps += 1
        b += 1
    secs = timers["oracle_s"]
    _ = oracle
    desc = (f"{nsteps} decoding steps (lookup+verify) round-robin over the 256 rollouts of RL "
            f"step 0, {timers.get('rows', 0)} logits rows, {tokens} tokens; oracle time only")
    return tokens / secs, desc, secs


# ---------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="q7")
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        log(f"note: WORLD_SIZE={world}, --gpus={args.gpus}")
    metric = "verified tokens/sec/GPU at V=151936, k=8; mean accepted length; HBM GB/s"
    unit = "verified tokens/s"
    workload = (f"{args.config}: V={cfg['V']}, {cfg['prompts'] * cfg['G']} rollouts/GPU "
                f"({cfg['prompts']} prompts x {cfg['G']}), k={cfg['k']}, lognormal lengths mean "
                f"{cfg['mean_len']} sigma {cfg['sigma']} cap {cfg['cap']}, T={cfg['T']}, "
                f"top_p={cfg['top_p']}, pools {cfg['G_pre']}/prompt, match rate "
                f"{cfg['match_rate']}")

    if args.impl == "reference":
        if rank != 0:
            return
        v, desc, secs = cpu_oracle_sample(cfg, args.cpu_budget / max(1, args.steps) * 1.0)
        # K steps of the bounded sample (each ~budget/K s of oracle time)
        vals = [v]
        for _ in range(1, args.steps):
            vals.append(cpu_oracle_sample(cfg, args.cpu_budget / max(1, args.steps))[0])
        val = float(np.median(vals))
        out = {"impl": "reference", "metric": metric, "value": val, "unit": unit,
               "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "u64", "data": "synthetic",
               "config": {"workload": workload},
               "cpu_baseline": {"value": val, "unit": unit, "cores": 1, "kind": "oracle",
                                "sample": desc},
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
    r = run_ours(args, cfg, rank, world, dist)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    st, rec = r["st"], r["rec"]
    V = cfg["V"]
    row_bytes = 2 * V
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if hbm else "fallback 6650 GB/s"
    hbm = hbm or 6650.0
    ms_per_step = r["elapsed_ms"] / args.steps
    value = r["tokens"] / (r["elapsed_ms"] / 1e3)
    # dominant kernel: the verify op (one cluster-kernel launch), timed by captured events
    vlaunches = rec["decode_steps"]
    v_avg_ms = rec["verify_ms"] / max(1, vlaunches)
    alg_bytes = rec["verify_rows_needed"] * row_bytes / max(1, vlaunches)   # per launch
    moved_bytes = rec["verify_rows_verified"] * row_bytes / max(1, vlaunches)
    achieved = alg_bytes / (v_avg_ms * 1e-3) / 1e9
    steady_alg = r["sst"]["rows_needed"] * row_bytes / (r["steady_ms"] * 1e-3) / 1e9
    steady_moved = r["sst"]["rows_verified"] * row_bytes / (r["steady_ms"] * 1e-3) / 1e9
    cpu = None
    if not args.no_cpu_baseline:
        cv, desc, secs = cpu_oracle_sample(cfg, args.cpu_budget)
        cpu = {"value": cv, "unit": unit, "cores": 1, "kind": "oracle", "sample": desc}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "verify_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("bytes_per_launch")
        except ValueError:
            traffic = None
    out = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded counter-hash bank of 8192 bf16 logit rows, perturbed pools)",
        "config": {"workload": workload, "parallelism": f"dp{args.gpus}",
                   "rollouts": cfg["prompts"] * cfg["G"] * args.gpus,
                   "l2": "inputs larger than L2 (2.5 GB logit bank, rows drawn by hash)",
                   "graph_chunk": args.chunk},
        "per_gpu_value": value / args.gpus,
        "acceptance_length": st["acceptance_length"], "draft_length": st["draft_length"],
        "acceptance_rate": st["acceptance_rate"], "decode_steps": st["decode_steps"],
        "tokens": int(r["tokens"]),
        "hbm_gbs": {"algorithmic": achieved, "moved": moved_bytes / (v_avg_ms * 1e-3) / 1e9,
                    "steady_algorithmic": steady_alg, "steady_moved": steady_moved},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic,
                     "kernel": "bs_verify_commit_lookup (verify_cluster_kernel: in-kernel plan, rows, "
                               "fused commit and next-draft lookup), avg over an instrumented replay "
                               "of the timed RL steps",
                     "peak_source": peak_src,
                     "steady_frac": steady_alg / hbm},
        "clocks": r["clocks"],
        "e2e": {"value": r["e2e_tokens"] / (r["e2e_ms"] / 1e3), "unit": unit,
                "h2d_bytes_per_step": r["e2e"]["h2d"], "d2h_bytes_per_step": r["e2e"]["d2h"]},
        "gpu_launches": rec["launches"],
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
