"""B200-native BubbleSpec hot path (arXiv 2605.08862): draft lookup over per-prompt pools
and lossless verification of model-free drafts, behind the C-ABI of include/bubblespec.h.

The CUDA library (libbubblespec.so, sm_100a) is required; there is no CPU fallback.
"""
from ._lib import LIB_PATH, BubbleSpecError, load  # noqa: F401
from .api import (  # noqa: F401
    BubbleSync,
    Context,
    bs_lm_head_logits,
    bs_route_plan,
    bs_unified_attention,
    bsx_synth_attn_values,
    bsx_synth_bank,
    nccl_comm_destroy,
    nccl_comm_init,
    nccl_unique_id,
)
from .engine import RolloutEngine  # noqa: F401
from .pregen import Pregenerator, pool_sequences  # noqa: F401
