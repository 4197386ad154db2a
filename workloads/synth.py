"""Counter-based synthetic inputs (numpy).  See workloads/__init__.py and DESIGN.md §5.

Every generator is a pure function of integer seeds and indices, built from the
32-bit ``lowbias32`` integer hash, so the CUDA twins in csrc/synth.cu reproduce
them bit for bit.  No value here depends on the method under test.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

M32 = 0xFFFFFFFF


def h32(x):
    """lowbias32 integer hash (C. Wellons), elementwise on uint32 arrays or ints."""
    x = np.asarray(x, dtype=np.uint32).copy()
    with np.errstate(over="ignore"):
        x ^= x >> np.uint32(16)
        x *= np.uint32(0x7FEB352D)
        x ^= x >> np.uint32(15)
        x *= np.uint32(0x846CA68B)
        x ^= x >> np.uint32(16)
    return x


def _mix(a, b):
    """h32(a ^ b) with b cast to uint32 (wrapping)."""
    b = np.asarray(b, dtype=np.int64).astype(np.uint32)
    return h32(np.asarray(a, dtype=np.uint32) ^ b)


def f32_to_bf16_bits(x):
    """Round-to-nearest-even fp32 -> bf16 bit pattern (finite inputs)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b):
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


LOGIT_SCALE = np.float32(0.015625)  # 2^-6: s in [-510, 510] -> logits in [-7.97, 7.97], sd 2.31


PEAK_GROUP = 16  # bank rows 16g .. 16g+15 share their peak column (same token, own noise)


def bank_peak(bank_seed: int, rows, V: int):
    """Peak (reference) column of each bank row: a function of the row's group of 16."""
    s = h32(np.uint32(bank_seed & M32) ^ np.uint32(0x5BD1E995))
    return (_mix(s, np.asarray(rows, dtype=np.int64) // PEAK_GROUP) % np.uint32(V)).astype(np.int32)


def bank_rows(bank_seed: int, rows, V: int, beta: float) -> np.ndarray:
    """bf16 bits [len(rows), V]: Irwin-Hall(4 bytes) noise * 2^-6; the peak column is beta."""
    rows = np.asarray(rows, dtype=np.int64)
    s0 = h32(np.uint32(bank_seed & M32))
    hr = _mix(s0, rows)[:, None]  # [R,1]
    cols = np.arange(V, dtype=np.uint32)[None, :]
    h = h32(hr ^ cols)
    s = ((h & 255) + ((h >> 8) & 255) + ((h >> 16) & 255) + (h >> 24)).astype(np.int32) - 510
    val = s.astype(np.float32) * LOGIT_SCALE
    peak = bank_peak(bank_seed, rows, V)
    val[np.arange(len(rows)), peak] = np.float32(beta)
    return f32_to_bf16_bits(val)


@dataclass(frozen=True)
class TargetSpec:
    """The synthetic target policy: which bank row is the distribution at a position.

    mode "position": row(P, t)        — peaked at the prompt's reference text R_P[t]
    mode "sample":   row(P, t, uid)   — like "position" (same peak R_P[t]), but each of a
                                        prompt's samples (uid mod 16) reads its own row of the
                                        peak group: no two rollouts share logits rows
    mode "markov":   row(P, prev)     — an order-1 Markov chain per prompt
    mode "mixed":    row(P, t, prev)  — depends on both (catches row/prefix misalignment)
    """

    V: int
    nbank: int
    bank_seed: int = 1
    target_seed: int = 2
    beta: float = 12.0
    mode: str = "position"


def target_row(spec: TargetSpec, P, t, prev, uid=0):
    """Bank row index of the target distribution for generated-token index t of a
    rollout (global id uid) of prompt P whose previous token is prev (vectorised)."""
    base = _mix(h32(np.uint32(spec.target_seed & M32)), P)
    if spec.mode == "sample":
        h = _mix(base, t)
        g = (h % np.uint32(spec.nbank // PEAK_GROUP)).astype(np.int64)
        return g * PEAK_GROUP + (np.asarray(uid, dtype=np.uint64) % np.uint64(PEAK_GROUP)).astype(np.int64)
    if spec.mode == "position":
        h = _mix(base, t)
    elif spec.mode == "markov":
        h = _mix(base, np.asarray(prev, dtype=np.int64) + 0x10000000)
    elif spec.mode == "mixed":
        h = _mix(_mix(base, t), np.asarray(prev, dtype=np.int64) + 0x10000000)
    else:
        raise ValueError(spec.mode)
    return (h % np.uint32(spec.nbank)).astype(np.int64)


def reference_text(spec: TargetSpec, P: int, length: int, prompt_last: int) -> np.ndarray:
    """R_P[t] = peak column of the target row at t when following the reference."""
    if spec.mode in ("position", "sample"):  # rows do not depend on the previous token
        r = target_row(spec, P, np.arange(length, dtype=np.int64), 0)
        return bank_peak(spec.bank_seed, r, spec.V).astype(np.int32)
    out = np.empty(length, dtype=np.int32)
    prev = prompt_last
    for t in range(length):
        r = target_row(spec, P, t, prev)
        out[t] = bank_peak(spec.bank_seed, np.array([r]), spec.V)[0]
        prev = int(out[t])
    return out


def prompt_tails(seed: int, prompt_ids, M: int, V: int) -> np.ndarray:
    """[n, M] random prompt tokens (all M positions valid)."""
    p = np.asarray(prompt_ids, dtype=np.int64)
    base = _mix(h32(np.uint32(seed & M32) ^ np.uint32(0x1234567)), p)[:, None]
    return (h32(base ^ np.arange(M, dtype=np.uint32)[None, :]) % np.uint32(V)).astype(np.int32)


def lognormal_lengths(seed: int, n: int, mean: float, sigma: float = 0.6, cap: int = 32768,
                      floor: int = 1) -> np.ndarray:
    """Lognormal response lengths with the given mean (mu = ln(mean) - sigma^2/2)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    mu = np.log(mean) - 0.5 * sigma * sigma
    x = rng.lognormal(mu, sigma, size=n)
    return np.clip(np.rint(x), floor, cap).astype(np.int32)


def make_pools(spec: TargetSpec, prompt_ids, tails: np.ndarray, G: int, seq_lens,
               match_rate: float, noise: float = 0.02, pool_seed: int = 3, prefix: int = 0,
               refs: dict | None = None):
    """Draft pools: per prompt, G copies of [last `prefix` prompt tokens] + R'_P where
    R'_P is the reference text with a SHARED substitution pattern at rate 1-match_rate
    plus independent per-copy noise at rate `noise`.

    Returns (seq_prompt int32 [n_seqs], seq_off int64 [n_seqs+1], tokens int32 [N]).
    seq_lens: [len(prompt_ids), G] response lengths of the pool sequences.
    """
    seq_lens = np.asarray(seq_lens, dtype=np.int64).reshape(len(prompt_ids), G)
    sub_thr = np.uint32(min(M32, int((1.0 - match_rate) * 4294967296.0)))
    noise_thr = np.uint32(min(M32, int(noise * 4294967296.0)))
    sp, offs, toks = [], [0], []
    s0 = h32(np.uint32(pool_seed & M32))
    for i, P in enumerate(prompt_ids):
        L = int(seq_lens[i].max()) if G else 0
        if refs is not None and P in refs:
            ref = refs[P][:L]
        else:
            ref = reference_text(spec, int(P), L, int(tails[i, -1]))
        t = np.arange(L, dtype=np.uint32)
        hp = _mix(s0, P)
        hs = h32(hp ^ t)
        shared = hs < sub_thr
        subst_tok = (h32(hs ^ np.uint32(0xA5A5A5A5)) % np.uint32(spec.V)).astype(np.int32)
        base = np.where(shared, subst_tok, ref)
        for g in range(G):
            hg = h32(_mix(hp, g + 1) ^ t)
            noisy = hg < noise_thr
            ntok = (h32(hg ^ np.uint32(0x3C3C3C3C)) % np.uint32(spec.V)).astype(np.int32)
            seq = np.where(noisy, ntok, base)[: seq_lens[i, g]]
            if prefix:
                seq = np.concatenate([tails[i, -prefix:], seq])
            sp.append(P)
            toks.append(seq.astype(np.int32))
            offs.append(offs[-1] + len(seq))
    tokens = np.concatenate(toks) if toks else np.zeros(0, np.int32)
    return (np.asarray(sp, dtype=np.int32), np.asarray(offs, dtype=np.int64), tokens)
