"""ctypes loader for libbubblespec.so (the C-ABI of include/bubblespec.h).

There is no fallback: if the CUDA library is missing this raises, loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbubblespec.so")
# profiling builds (e.g. libbubblespec_timing.so, -DBS_PHASE_TIMING) are selected explicitly
if os.environ.get("BS_LIB_VARIANT"):
    LIB_PATH = os.path.join(_HERE, f"libbubblespec_{os.environ['BS_LIB_VARIANT']}.so")

BS_OK, BS_ERR_INVALID, BS_ERR_OOM, BS_ERR_CUDA, BS_ERR_STALE, BS_ERR_CAPACITY, BS_ERR_NCCL, \
    BS_ERR_DEVICE = range(8)
STATUS_NAMES = ["BS_OK", "BS_ERR_INVALID", "BS_ERR_OOM", "BS_ERR_CUDA", "BS_ERR_STALE",
                "BS_ERR_CAPACITY", "BS_ERR_NCCL", "BS_ERR_DEVICE"]


class bs_config(C.Structure):
    _fields_ = [("vocab", C.c_int32), ("eos_id", C.c_int32), ("k_max", C.c_int32),
                ("match_max", C.c_int32), ("match_min", C.c_int32), ("max_rollouts", C.c_int32),
                ("pool_capacity_tokens", C.c_int64), ("pool_capacity_seqs", C.c_int32),
                ("device", C.c_int32), ("seed", C.c_uint64)]


class bs_sampling(C.Structure):
    _fields_ = [("temperature", C.c_float), ("top_p", C.c_float), ("top_k", C.c_int32)]


_V = C.c_void_p
_I32, _I64, _U64, _U32 = C.c_int32, C.c_int64, C.c_uint64, C.c_uint32

# name -> (restype, argtypes); the list mirrors include/bubblespec.h
SIGNATURES = {
    "bs_create": (C.c_int, [C.POINTER(bs_config), C.POINTER(_V)]),
    "bs_destroy": (None, [_V]),
    "bs_last_error": (C.c_char_p, [_V]),
    "bs_sync_status": (C.c_int, [_V, _V, C.POINTER(_U32)]),
    "bs_version": (C.c_char_p, []),
    "bs_rollout_begin": (C.c_int, [_V, _I32, _V, _V, _V, _V, _V, _V]),
    "bs_rollout_state": (C.c_int, [_V, _I32, _V, _V, _V, _V]),
    "bs_rollout_live": (C.c_int, [_V, _I32, _V, _V, _V]),
    "bs_draft_pool_put": (C.c_int, [_V, _U64, _I32, _V, _V, _V, _I64, _V]),
    "bs_draft_pool_seal": (C.c_int, [_V, _U64, _V]),
    "bs_draft_exchange": (C.c_int, [_V, _V, _I32, _I32, _U64, _V]),
    "bs_route_plan": (C.c_int, [_I32, _I32, _V, _V, _V, _I64, _I64, _V, _V, _V, _V, _V, _V]),
    "bs_nccl_unique_id": (C.c_int, [_V]),
    "bs_nccl_comm_init": (C.c_int, [C.POINTER(_V), _V, _I32, _I32]),
    "bs_nccl_comm_destroy": (C.c_int, [_V]),
    "bs_draft_lookup": (C.c_int, [_V, _U64, _I32, _V, _I32, _V, _V, _V, _V]),
    "bs_verify_step": (C.c_int, [_V, _I32, _V, _V, _V, _I64, _V, _V, _I32, bs_sampling, _V, _V,
                                 _V, _V, _V, _V]),
    "bs_bubble_sync_create": (C.c_int, [_I32, C.POINTER(_V)]),
    "bs_bubble_sync_export": (C.c_int, [_V, _V]),
    "bs_bubble_sync_open": (C.c_int, [_I32, _V, C.POINTER(_V)]),
    "bs_bubble_sync_destroy": (None, [_V]),
    "bs_bubble_sync_arrive": (C.c_int, [_V, _I32, _U64, _V]),
    "bs_bubble_sync_poll": (C.c_int, [_V, _I32, _U64, _V, _V]),
    "bs_unified_attention_workspace": (C.c_int, [_I32, _V, _V, _I32, _I32, C.POINTER(_I64)]),
    "bs_unified_attention": (C.c_int, [_V, _V, _V, _I64, _V, _I32, _V, _V, _V, _I32, _I32, _I32, _I32, _I32,
                                       C.c_float, _V, _V, _I64, _V]),
    "bsx_synth_attn_values": (C.c_int, [_V, _I64, _U32, C.c_float, _V]),
    "bs_lm_head_logits": (C.c_int, [_V, _V, _I32, _I32, _I32, _V, _I64, _V, _V, _V]),
    "bsx_set_row_stats": (C.c_int, [_V, _V, _V]),
    "bs_draft_lookup_ngram": (C.c_int, [_V, _U64, _I32, _V, _I32, _I32, _I32, _V, _V, _V, _V]),
    "bs_draft_set_min_token_prob": (C.c_int, [_V, C.c_float]),
    "bs_verify_commit": (C.c_int, [_V, _I32, _V, _V, _V, _I64, _V, _V, _I32, bs_sampling, _V, _V,
                                   _V, _V, _V, _V, _V]),
    "bs_verify_commit_lookup": (C.c_int, [_V, _U64, _I32, _V, _V, _V, _I64, _V, _V, _I32, bs_sampling, _V,
                                          _V, _V, _V, _V, _V, _V, _V]),
    "bs_commit": (C.c_int, [_V, _I32, _V, _V, _V, _I32, _V, _V]),
    "bs_stats_read": (C.c_int, [_V, _V, _I32, _I32, _V]),
    "bs_rollout_bind_output": (C.c_int, [_V, _V, _I64]),
    "bsx_set_verify_kernel": (C.c_int, [_V, _I32]),
    "bsx_set_early_plan": (C.c_int, [_V, _I32]),
    "bsx_set_max_clusters": (C.c_int, [_V, _I32]),
    "bsx_launch_info": (C.c_int, [_V, C.POINTER(C.c_int64), _I32]),
    "bsx_synth_bank": (C.c_int, [_V, _I64, _I32, _U32, C.c_float, _V]),
    "bsx_target_rows": (C.c_int, [_V, _I32, _V, _V, _V, _I32, _U32, _I32, _I64, _V, _V]),
}

_lib = None


def load():
    """Load the CUDA library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libbubblespec.so not found at {LIB_PATH}: the CUDA extension is required "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
        lib = C.CDLL(LIB_PATH)
        if hasattr(lib, "bsx_phase_times"):  # diagnostics (not part of the C-ABI header)
            lib.bsx_phase_times.restype = C.c_int
            lib.bsx_phase_times.argtypes = [C.c_void_p, C.c_int]
        if hasattr(lib, "bsx_trace_read"):
            lib.bsx_trace_read.restype = C.c_int
            lib.bsx_trace_read.argtypes = [C.c_void_p, C.c_int, C.c_int]
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class BubbleSpecError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str = ""):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{where}: {name}{': ' + msg if msg else ''}")
