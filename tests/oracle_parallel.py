"""Run the oracle's Alg. 1 loop (oracle/rollout.py) over many rollouts on all host cores.

TEST INFRASTRUCTURE ONLY.  Rollouts are independent given the pools, so they are
split by prompt over forked worker processes; each worker runs the plain oracle exactly as
``oracle.rollout.run_rollouts`` does, one rollout after another.  The workers never touch
CUDA (numpy + the C oracle only), so forking a process that holds a CUDA context is safe.
"""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

_JOB = {}


def _run_group(bs):
    from oracle.rollout import OracleRollout, bank_row_fn, pools_by_prompt, run_rollouts

    j = _JOB
    pools = pools_by_prompt(j["seq_prompt"], j["seq_off"], j["tokens"])
    ros = [OracleRollout(prompt=int(j["pid"][b]), uid=int(j["uids"][b]),
                         context=[int(x) for x in j["tails"][b] if x >= 0], max_len=int(j["max_len"][b]))
           for b in bs]
    run_rollouts(ros, pools, bank_row_fn(j["spec"]), k=j["k"], M=j["M"], Lmin=1, T=j["T"],
                 top_p=j["top_p"], seed=j["seed"], eos=j["eos"], max_steps=j["max_steps"])
    out = []
    for b, ro in zip(bs, ros):
        steps = [(q, len(emitted), acc) for (q, _m, _d, emitted, acc, _o) in ro.steps]
        out.append((b, ro.generated, steps))
    return out


def run_oracle_parallel(inp: dict, *, k, M, T, top_p, seed, eos, max_steps, procs=None):
    """inp: seq_prompt, seq_off, tokens, pid, tails, uids, max_len, spec (numpy / TargetSpec).
    Returns {rollout: (generated tokens, [(q, emitted, accepted) per step])}."""
    _JOB.clear()
    _JOB.update(inp)
    _JOB.update(k=k, M=M, T=T, top_p=top_p, seed=seed, eos=eos, max_steps=max_steps)
    n = len(inp["pid"])
    # group rollouts by prompt (a worker's row cache then serves the whole group)
    order = np.argsort(np.asarray(inp["pid"]), kind="stable")
    procs = procs or max(1, min(os.cpu_count() or 1, 64))
    groups = [list(map(int, g)) for g in np.array_split(order, min(n, procs * 2)) if len(g)]
    ctx = mp.get_context("fork")
    with ctx.Pool(min(procs, len(groups))) as pool:
        res = pool.map(_run_group, groups, chunksize=1)
    out = {}
    for part in res:
        for b, gen, steps in part:
            out[b] = (gen, steps)
    return out


def oracle_counters(res: dict, nbins: int = 33):
    """The device statistics counters (bs_stats_read order) of an oracle run."""
    c = np.zeros(8 + nbins, dtype=np.int64)
    for _gen, steps in res.values():
        for q, emitted, acc in steps:
            if q >= 1:
                c[0] += 1
                c[2] += emitted
                c[4] += acc
                c[5] += q
                c[8 + emitted] += 1
            else:
                c[1] += 1
                c[3] += emitted
    return c
