"""Seeded synthetic inputs of the unified variable-query-length decode attention (SURVEY
§8(f)2; Table 2 at P:220-232): a batch of requests, each with a context of
ctx_len tokens whose K/V already sit in a paged cache, the last q_len of them being the
step's query tokens (1 for a plain decode, 1 + drafts for a speculative request).

Holds no attention arithmetic: only bf16 values (counter hashes), the page assignment and the
layouts.  Layout of the paged cache ("f2"): K and V are each
[num_pages, H_kv, PAGE, d] bf16 (a page holds PAGE consecutive tokens of one request, all KV
heads, each head's PAGE x d block contiguous, d contiguous); page_table[b, i] is the page of
tokens [i*PAGE, (i+1)*PAGE) of request b; queries are [sum_b q_len_b, H_q, d] bf16 with
request b's tokens at rows q_off[b] .. q_off[b+1]).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .synth import f32_to_bf16_bits, h32

PAGE = 64


@dataclass
class AttnBatch:
    q: np.ndarray            # uint16 bf16 bits [T, H_q, d]
    k_cache: np.ndarray      # uint16 [num_pages, H_kv, PAGE, d]
    v_cache: np.ndarray      # uint16 [num_pages, H_kv, PAGE, d]
    page_table: np.ndarray   # int32 [B, max_pages]
    ctx_len: np.ndarray      # int32 [B]
    q_off: np.ndarray        # int32 [B + 1]
    H_q: int
    H_kv: int
    d: int


def _vals(seed: int, salt: int, n: int, scale: float) -> np.ndarray:
    """n hashed values, approximately N(0, scale^2) (sum of 4 hashed bytes)."""
    i = np.arange(n, dtype=np.uint64)
    u = h32((i * np.uint64(0x9E3779B1) + np.uint64(seed * 1000003 + salt)) & np.uint64(0xFFFFFFFF))
    u = u.astype(np.uint32)
    s = ((u & 0xFF) + ((u >> 8) & 0xFF) + ((u >> 16) & 0xFF) + (u >> 24)).astype(np.float32) - 510.0
    return (s * np.float32(scale / 147.8)).astype(np.float32)


def make_attn_batch(seed: int, q_len, ctx_len, H_q: int = 28, H_kv: int = 4, d: int = 128,
                    shuffle_pages: bool = True, spare_pages: int = 3) -> AttnBatch:
    """Requests b with q_len[b] query tokens (the last ones of its ctx_len[b]-token context).
    Pages are assigned in a seeded random order (so paging is exercised), plus spare pages
    that no request uses."""
    q_len = np.asarray(q_len, dtype=np.int32)
    ctx_len = np.asarray(ctx_len, dtype=np.int32)
    B = len(q_len)
    assert (q_len >= 1).all() and (ctx_len >= q_len).all()
    npg = (ctx_len + PAGE - 1) // PAGE
    total = int(npg.sum()) + spare_pages
    rng = np.random.default_rng(seed)
    order = rng.permutation(total) if shuffle_pages else np.arange(total)
    maxp = max(1, int(npg.max()))
    page_table = np.full((B, maxp), -1, dtype=np.int32)
    c = 0
    for b in range(B):
        page_table[b, : npg[b]] = order[c:c + npg[b]]
        c += npg[b]
    k = _vals(seed, 1, total * H_kv * PAGE * d, 1.0).reshape(total, H_kv, PAGE, d)
    v = _vals(seed, 2, total * H_kv * PAGE * d, 1.0).reshape(total, H_kv, PAGE, d)
    q_off = np.zeros(B + 1, dtype=np.int32)
    q_off[1:] = np.cumsum(q_len)
    q = _vals(seed, 3, int(q_off[-1]) * H_q * d, 1.0).reshape(int(q_off[-1]), H_q, d)
    return AttnBatch(q=f32_to_bf16_bits(q), k_cache=f32_to_bf16_bits(k), v_cache=f32_to_bf16_bits(v),
                     page_table=page_table, ctx_len=ctx_len, q_off=q_off, H_q=H_q, H_kv=H_kv, d=d)


def logical_kv(batch: AttnBatch, b: int):
    """Request b's K and V as logical [ctx_len, H_kv, d] bf16-bit arrays (gathered from its
    pages): the paging is input plumbing, not attention arithmetic."""
    L = int(batch.ctx_len[b])
    npg = (L + PAGE - 1) // PAGE
    pages = batch.page_table[b, :npg]
    k = batch.k_cache[pages].transpose(0, 2, 1, 3).reshape(npg * PAGE, batch.H_kv, batch.d)[:L]
    v = batch.v_cache[pages].transpose(0, 2, 1, 3).reshape(npg * PAGE, batch.H_kv, batch.d)[:L]
    return k, v
