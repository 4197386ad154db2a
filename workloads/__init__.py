"""Seeded synthetic workload generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no softmax, no acceptance test,
no lookup): it only produces inputs — bf16 logit rows, the synthetic target's
row-selection rule, reference texts, draft pools and response lengths — from
counter-based integer hashes, so that the numpy generators here and their CUDA
twins (``bsx_synth_bank`` / ``bsx_target_rows`` in the product library) produce
bit-identical data.  Recipe: DESIGN.md §5 ("synthetic inputs").
"""
from .synth import (  # noqa: F401
    h32,
    f32_to_bf16_bits,
    bf16_bits_to_f32,
    bank_rows,
    bank_peak,
    target_row,
    reference_text,
    make_pools,
    prompt_tails,
    lognormal_lengths,
    TargetSpec,
)
