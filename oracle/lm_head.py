"""LM-head logits and their row statistics — TEST INFRASTRUCTURE ONLY (parity oracle of
SURVEY §8(f)3, the LM-head GEMM whose epilogue also emits what the verify's first pass needs).

logits[r, v] = bf16( sum_k h[r, k] * W[v, k] )   (the target policy's logits: "the
actual decoding distribution used by the target policy" starts from them), computed in fp64 and
rounded once to bf16 (round to nearest even); the row statistics are readings R0/R1 of the
verify: the row maximum of the bf16 logits, the lowest index attaining it, and whether any
logit is NaN / +inf.  numpy's fp64 matmul is the one library step.  Pins:
tests/test_attention_oracle.py::test_lm_head_*.
"""
from __future__ import annotations

import numpy as np


def _f64(bits):
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def _bf16_rne(x64):
    """fp64 -> bf16 bits, round to nearest even (finite values), via the exact fp32 value when
    it is representable, else through the bit pattern of the fp64 value."""
    x = np.asarray(x64, dtype=np.float64)
    # round fp64 to bf16 directly: 8 mantissa bits kept of 52
    b = x.view(np.uint64)
    sign = (b >> np.uint64(63)) & np.uint64(1)
    mag = b & np.uint64(0x7FFFFFFFFFFFFFFF)
    lsb = (mag >> np.uint64(45)) & np.uint64(1)
    rounded = (mag + np.uint64(0x0FFFFFFFFFFF) + lsb) >> np.uint64(45)  # 52 - 7 = 45 bits dropped
    # rounded holds the fp64 exponent (11 bits) and 7 mantissa bits; rebuild as fp64 then take the
    # fp32 bit pattern's top half (exact: the value has <= 8 significant bits)
    y = ((rounded << np.uint64(45)) | (sign << np.uint64(63))).view(np.float64)
    return (y.astype(np.float32).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def lm_head_logits(h_bits, w_bits):
    """h [rows, d], W [V, d] (bf16 bits) -> logits [rows, V] (bf16 bits)."""
    return _bf16_rne(_f64(h_bits) @ _f64(w_bits).T)


def row_stats(logit_bits):
    """Per row: (max as fp32, lowest argmax, bad) of bf16 logits (readings R0, R1)."""
    x = _f64(logit_bits)
    bad = ~np.isfinite(x) & ~((x == -np.inf))
    m = np.where(np.isnan(x), -np.inf, x).max(axis=1)
    am = np.argmax(x == m[:, None], axis=1)
    return m.astype(np.float32), am.astype(np.int64), bad.any(axis=1)
