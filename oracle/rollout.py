"""Alg. 1's rollout loop driven step by step through the C oracle.

TEST INFRASTRUCTURE ONLY.  Each decoding step of a rollout is: draft lookup from
the prompt's pool (brute force) -> the synthetic target's rows for positions
pos..pos+q -> ``verify_one`` (Alg. 1 step + bonus) -> commit (append the emitted
tokens; finished on EOS or max_len; reading L6 / P:530 "while |y| < L and not EOS").
Rollouts are independent given the pools, so they are run one after another.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np


@dataclass
class OracleRollout:
    prompt: int
    uid: int
    context: list          # prompt tail tokens followed by generated tokens
    max_len: int
    pos: int = 0           # generated tokens so far
    finished: bool = False
    generated: list = field(default_factory=list)
    steps: list = field(default_factory=list)  # (q, m_star, draft, emitted, accepted)


def pools_by_prompt(seq_prompt, seq_off, tokens):
    pools = {}
    for s, P in enumerate(seq_prompt):
        pools.setdefault(int(P), []).append([int(x) for x in tokens[seq_off[s]:seq_off[s + 1]]])
    return pools


def step(ro: OracleRollout, pools: dict, row_fn, *, k: int, M: int, Lmin: int, T: float,
         top_p: float, seed: int, eos: int, timers: dict | None = None, top_k: int = 0,
         ngram: tuple | None = None, min_token_prob: float = 0.0):
    """One decoding step of one rollout.  row_fn(P, positions, prevs, uid) -> list of bf16 rows.
    ngram = (n_min, n_max): draft with the n-gram linear-scan drafter (reading N1) instead of
    the suffix lookup; min_token_prob > 0: confidence-scored suffix drafts (reading C1)."""
    from . import lookup, lookup_ngram, verify_one

    if ro.finished or ro.pos >= ro.max_len:
        return None
    t0 = time.perf_counter()
    if ngram is None:
        draft, mstar = lookup(pools.get(ro.prompt, []), ro.context[-M:], M, Lmin, k, min_token_prob)
    else:
        draft, mstar = lookup_ngram(pools.get(ro.prompt, []), ro.context[-M:], ngram[0], ngram[1], k)
    q = min(len(draft), k, max(0, ro.max_len - ro.pos - 1))
    draft = draft[:q]
    t1 = time.perf_counter()
    prevs = [ro.context[-1]] + draft
    rows = row_fn(ro.prompt, [ro.pos + j for j in range(q + 1)], prevs, ro.uid)
    t2 = time.perf_counter()
    out = verify_one(rows, T, top_p, seed, ro.uid, ro.pos, ro.max_len, eos, ro.finished, draft, k,
                     top_k=top_k)
    t3 = time.perf_counter()
    if timers is not None:
        timers["oracle_s"] = timers.get("oracle_s", 0.0) + (t1 - t0) + (t3 - t2)
        timers["rows"] = timers.get("rows", 0) + out.rows_used
    ro.context.extend(out.tokens)
    ro.generated.extend(out.tokens)
    ro.pos += len(out.tokens)
    if (eos >= 0 and out.tokens and out.tokens[-1] == eos) or ro.pos >= ro.max_len:
        ro.finished = True
    ro.steps.append((q, mstar, draft, out.tokens, out.accepted, out))
    return out


def run_rollouts(rollouts, pools, row_fn, *, k, M, Lmin, T, top_p, seed, eos, max_steps=None,
                 timers=None, top_k=0, ngram=None, min_token_prob=0.0):
    for ro in rollouts:
        n = 0
        while not ro.finished and (max_steps is None or n < max_steps):
            step(ro, pools, row_fn, k=k, M=M, Lmin=Lmin, T=T, top_p=top_p, seed=seed, eos=eos,
                 timers=timers, top_k=top_k, ngram=ngram, min_token_prob=min_token_prob)
            n += 1
    return rollouts


def bank_row_fn(spec, cache: dict | None = None):
    """row_fn over the synthetic bank (workloads.TargetSpec)."""
    from workloads import bank_rows, target_row

    cache = {} if cache is None else cache

    def fn(P, positions, prevs, uid=0):
        idx = target_row(spec, np.full(len(positions), P), np.asarray(positions),
                         np.asarray(prevs), np.uint64(uid))
        out = []
        if len(cache) > 2048:  # bounded: with per-rollout rows ("sample" mode) few rows repeat
            cache.clear()
        for r in idx:
            r = int(r)
            if r not in cache:
                cache[r] = bank_rows(spec.bank_seed, [r], spec.V, spec.beta)[0]
            out.append(cache[r])
        return out

    return fn
