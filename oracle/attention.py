"""Unified variable-query-length decode attention — TEST INFRASTRUCTURE ONLY (the parity
oracle of SURVEY §8(f)2).  Plain numpy in fp64, one request, one query head, one query token
at a time; shares no code with the CUDA path.

What it computes (one operator for "normal and decode queries" with "variable query
lengths within a short range"; the attention itself is the standard causal softmax attention
of the target model): for request b with context length L_b whose last q_b tokens are the
step's queries (the decode token and the drafts being verified), query token i (0 <= i < q_b)
sits at absolute position p = L_b - q_b + i and attends the keys at positions 0..p (causal):

    o[b, i, h] = sum_{j <= p} softmax_j( q[b, i, h] . k[b, j, h // G] * scale ) v[b, j, h // G]

with G = H_q / H_kv query heads per KV head (grouped-query attention) and scale = 1/sqrt(d)
unless given.  Inputs are bf16 bit patterns (converted exactly to fp64); the result is fp64.
Pins: tests/test_attention_oracle.py.
"""
from __future__ import annotations

import numpy as np


def _f64(bits):
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def attention_request(q_bits, k_bits, v_bits, H_kv: int, scale: float | None = None):
    """One request: q [q_len, H_q, d], k / v [L, H_kv, d] (bf16 bits, logical order).
    Returns o [q_len, H_q, d] in fp64."""
    q, k, v = _f64(q_bits), _f64(k_bits), _f64(v_bits)
    q_len, H_q, d = q.shape
    L = k.shape[0]
    G = H_q // H_kv
    sc = 1.0 / np.sqrt(d) if scale is None else scale
    o = np.zeros((q_len, H_q, d), dtype=np.float64)
    for i in range(q_len):
        p = L - q_len + i                     # absolute position of query token i
        for h in range(H_q):
            kv = h // G
            s = k[: p + 1, kv, :] @ q[i, h, :] * sc   # logits of keys 0..p
            w = np.exp(s - s.max())
            w /= w.sum()
            o[i, h, :] = w @ v[: p + 1, kv, :]
    return o


def attention_batch(batch, scale: float | None = None):
    """Every request of a workloads.attn.AttnBatch: o [T, H_q, d] fp64 in query-row order."""
    from workloads.attn import logical_kv

    out = np.zeros(batch.q.shape, dtype=np.float64)
    for b in range(len(batch.ctx_len)):
        k, v = logical_kv(batch, b)
        r0, r1 = int(batch.q_off[b]), int(batch.q_off[b + 1])
        out[r0:r1] = attention_request(batch.q[r0:r1], k, v, batch.H_kv, scale)
    return out
