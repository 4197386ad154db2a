"""Thin Python binding of the C-ABI (include/bubblespec.h): argument marshalling only.

Every function has the name of the C call it wraps and passes torch CUDA tensors as raw
device pointers; every step of the hot path runs in libbubblespec.so's kernels.  PyTorch
provides device memory and streams only.
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import BubbleSpecError, bs_config, bs_sampling, load

_V = C.c_void_p


def _p(t):
    """Device pointer of a tensor (or None)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return _V(t.data_ptr())


def _stream(stream, device):
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return _V(s.cuda_stream)


def _chk(ctx, st, where):
    if st != 0:
        msg = load().bs_last_error(ctx.handle if ctx is not None else None)
        raise BubbleSpecError(st, where, msg.decode() if msg else "")


class Context:
    """Owns a bs_ctx (pools, index, rollout slots, scratch) on one GPU."""

    def __init__(self, vocab: int, eos_id: int = -1, k_max: int = 8, match_max: int = 32,
                 match_min: int = 1, max_rollouts: int = 256, pool_capacity_tokens: int = 1 << 20,
                 pool_capacity_seqs: int = 1 << 14, device: int | None = None, seed: int = 0):
        lib = load()
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        self.vocab, self.eos_id, self.k_max, self.M = vocab, eos_id, k_max, match_max
        self.match_min, self.max_rollouts, self.seed = match_min, max_rollouts, seed
        cfg = bs_config(vocab, eos_id, k_max, match_max, match_min, max_rollouts,
                        pool_capacity_tokens, pool_capacity_seqs, device, seed)
        h = _V()
        st = lib.bs_create(C.byref(cfg), C.byref(h))
        if st != 0:
            raise BubbleSpecError(st, "bs_create", (lib.bs_last_error(None) or b"").decode())
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            load().bs_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ C calls
    def bs_sync_status(self, stream=None) -> int:
        w = C.c_uint32(0)
        st = load().bs_sync_status(self.handle, _stream(stream, self.device), C.byref(w))
        if st not in (0, 4, 7):  # OK, STALE (BS_DEV_STALE), DEVICE: the word says which
            _chk(self, st, "bs_sync_status")
        return int(w.value)

    def bs_rollout_begin(self, slots, uids, prompt_ids, prompt_tail, max_len, stream=None):
        n = slots.numel()
        _chk(self, load().bs_rollout_begin(self.handle, n, _p(slots), _p(uids), _p(prompt_ids),
                                           _p(prompt_tail), _p(max_len),
                                           _stream(stream, self.device)), "bs_rollout_begin")

    def bs_rollout_live(self, slots, live, stream=None):
        _chk(self, load().bs_rollout_live(self.handle, slots.numel(), _p(slots), _p(live),
                                          _stream(stream, self.device)), "bs_rollout_live")

    def bs_rollout_state(self, slots, pos=None, finished=None, stream=None):
        _chk(self, load().bs_rollout_state(self.handle, slots.numel(), _p(slots), _p(pos),
                                           _p(finished), _stream(stream, self.device)),
             "bs_rollout_state")

    def bs_draft_pool_put(self, rl_step, prompt_ids, seq_offsets, tokens, n_tokens: int,
                          stream=None):
        _chk(self, load().bs_draft_pool_put(self.handle, rl_step, prompt_ids.numel(),
                                            _p(prompt_ids), _p(seq_offsets), _p(tokens),
                                            n_tokens, _stream(stream, self.device)),
             "bs_draft_pool_put")

    def bs_draft_set_min_token_prob(self, min_token_prob: float):
        _chk(self, load().bs_draft_set_min_token_prob(self.handle, float(min_token_prob)),
             "bs_draft_set_min_token_prob")

    def bs_draft_pool_seal(self, rl_step, stream=None):
        _chk(self, load().bs_draft_pool_seal(self.handle, rl_step, _stream(stream, self.device)),
             "bs_draft_pool_seal")

    def bs_draft_exchange(self, comm, rank: int, world: int, rl_step, stream=None):
        _chk(self, load().bs_draft_exchange(self.handle, comm, rank, world, rl_step,
                                            _stream(stream, self.device)), "bs_draft_exchange")

    def bs_draft_lookup(self, rl_step, slots, k, draft_tokens, draft_len, match_len=None,
                        stream=None):
        _chk(self, load().bs_draft_lookup(self.handle, rl_step, slots.numel(), _p(slots), k,
                                          _p(draft_tokens), _p(draft_len), _p(match_len),
                                          _stream(stream, self.device)), "bs_draft_lookup")

    def bs_draft_lookup_ngram(self, rl_step, slots, k, n_min, n_max, draft_tokens, draft_len,
                              match_len=None, stream=None):
        _chk(self, load().bs_draft_lookup_ngram(self.handle, rl_step, slots.numel(), _p(slots), k, n_min,
                                                n_max, _p(draft_tokens), _p(draft_len), _p(match_len),
                                                _stream(stream, self.device)), "bs_draft_lookup_ngram")

    def bs_verify_step(self, slots, logits, row_index, row_stride, draft_tokens, draft_len, k,
                       temperature, top_p, out_tokens, out_len, out_accepted, out_norm=None,
                       out_z=None, stream=None, top_k=0):
        sp = bs_sampling(temperature, top_p, top_k)
        _chk(self, load().bs_verify_step(self.handle, slots.numel(), _p(slots), _p(logits),
                                         _p(row_index), row_stride, _p(draft_tokens),
                                         _p(draft_len), k, sp, _p(out_tokens), _p(out_len),
                                         _p(out_accepted), _p(out_norm), _p(out_z),
                                         _stream(stream, self.device)), "bs_verify_step")

    def bs_verify_commit(self, slots, logits, row_index, row_stride, draft_tokens, draft_len, k,
                         temperature, top_p, out_tokens, out_len, out_accepted, finished=None,
                         out_norm=None, out_z=None, stream=None, top_k=0):
        sp = bs_sampling(temperature, top_p, top_k)
        _chk(self, load().bs_verify_commit(self.handle, slots.numel(), _p(slots), _p(logits),
                                           _p(row_index), row_stride, _p(draft_tokens),
                                           _p(draft_len), k, sp, _p(out_tokens), _p(out_len),
                                           _p(out_accepted), _p(out_norm), _p(out_z), _p(finished),
                                           _stream(stream, self.device)), "bs_verify_commit")

    def bs_verify_commit_lookup(self, rl_step, slots, logits, row_index, row_stride, draft_tokens,
                                draft_len, k, temperature, top_p, out_tokens, out_len, out_accepted,
                                finished=None, match_len=None, out_norm=None, out_z=None, stream=None,
                                top_k=0):
        """bs_verify_commit, then this step's commit feeds the next step's draft lookup in the
        same launch: draft_tokens / draft_len are overwritten with the next step's drafts."""
        sp = bs_sampling(temperature, top_p, top_k)
        _chk(self, load().bs_verify_commit_lookup(self.handle, rl_step, slots.numel(), _p(slots), _p(logits),
                                                  _p(row_index), row_stride, _p(draft_tokens),
                                                  _p(draft_len), k, sp, _p(out_tokens), _p(out_len),
                                                  _p(out_accepted), _p(out_norm), _p(out_z), _p(finished),
                                                  _p(match_len), _stream(stream, self.device)),
             "bs_verify_commit_lookup")

    def bs_commit(self, slots, out_tokens, out_len, k, finished=None, stream=None):
        _chk(self, load().bs_commit(self.handle, slots.numel(), _p(slots), _p(out_tokens),
                                    _p(out_len), k, _p(finished), _stream(stream, self.device)),
             "bs_commit")

    def bs_stats_read(self, reset: bool = False, stream=None):
        import numpy as np

        out = np.zeros(41, dtype=np.uint64)
        _chk(self, load().bs_stats_read(self.handle, _V(out.ctypes.data), 41, int(reset),
                                        _stream(stream, self.device)), "bs_stats_read")
        return out

    def bs_rollout_bind_output(self, responses=None, stride: int = 0):
        _chk(self, load().bs_rollout_bind_output(self.handle, _p(responses),
                                                 stride if responses is not None else 0),
             "bs_rollout_bind_output")

    VERIFY_KERNELS = {"auto": 0, "rows": 1, "cluster": 3}

    def bsx_set_verify_kernel(self, kind):
        kind = self.VERIFY_KERNELS[kind] if isinstance(kind, str) else int(kind)
        _chk(self, load().bsx_set_verify_kernel(self.handle, kind), "bsx_set_verify_kernel")

    def bsx_launch_info(self) -> dict:
        out = (C.c_int64 * 4)()
        load().bsx_launch_info(self.handle, out, 4)
        return {"clusters": int(out[0]), "cooperative": int(out[1]), "sms": int(out[2]),
                "early_plan": int(out[3])}

    def bsx_set_early_plan(self, on: bool):
        _chk(self, load().bsx_set_early_plan(self.handle, int(bool(on))), "bsx_set_early_plan")

    def bsx_set_row_stats(self, row_key=None, row_bad=None):
        _chk(self, load().bsx_set_row_stats(self.handle, _p(row_key), _p(row_bad)), "bsx_set_row_stats")

    def bsx_set_max_clusters(self, max_clusters: int):
        _chk(self, load().bsx_set_max_clusters(self.handle, int(max_clusters)), "bsx_set_max_clusters")

    def bsx_target_rows(self, slots, draft_tokens, draft_len, k, target_seed, mode, nbank,
                        row_index, stream=None):
        _chk(self, load().bsx_target_rows(self.handle, slots.numel(), _p(slots), _p(draft_tokens),
                                          _p(draft_len), k, target_seed, mode, nbank,
                                          _p(row_index), _stream(stream, self.device)),
             "bsx_target_rows")


def bsx_synth_bank(bank, rows: int, V: int, bank_seed: int, beta: float, stream=None):
    st = load().bsx_synth_bank(_p(bank), rows, V, bank_seed & 0xFFFFFFFF, beta,
                               _stream(stream, bank.device))
    _chk(None, st, "bsx_synth_bank")


def bs_route_plan(world, rank, counts, offs_all, prompts_all, max_seqs, max_tokens):
    """Host routing plan (numpy in/out); see include/bubblespec.h."""
    import numpy as np

    counts = np.ascontiguousarray(counts, dtype=np.int64)
    offs_all = np.ascontiguousarray(offs_all, dtype=np.int64)
    prompts_all = np.ascontiguousarray(prompts_all, dtype=np.int32)
    tot = int(counts[0::2].sum()) + 1
    src, dst, ln = (np.zeros(tot, np.int64) for _ in range(3))
    pr = np.zeros(tot, np.int32)
    nk, nt = C.c_int32(), C.c_int64()
    pp = lambda a: _V(a.ctypes.data)  # noqa: E731
    rc = load().bs_route_plan(world, rank, pp(counts), pp(offs_all), pp(prompts_all), max_seqs,
                              max_tokens, pp(src), pp(dst), pp(ln), pp(pr), C.byref(nk),
                              C.byref(nt))
    if rc != 0:
        raise ValueError("inconsistent routing metadata")
    k = nk.value
    return src[:k], dst[:k], ln[:k], pr[:k], int(nt.value)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _chk(None, load().bs_nccl_unique_id(buf), "bs_nccl_unique_id")
    return buf.raw


def nccl_comm_init(uid: bytes, world: int, rank: int):
    comm = _V()
    buf = C.create_string_buffer(uid, 128)
    _chk(None, load().bs_nccl_comm_init(C.byref(comm), buf, world, rank), "bs_nccl_comm_init")
    return comm


def nccl_comm_destroy(comm):
    _chk(None, load().bs_nccl_comm_destroy(comm), "bs_nccl_comm_destroy")


class BubbleSync:
    """The polling synchronizer of pre-generation (bs_bubble_sync_*).  The owner
    rank creates it (handle=None) and sends export() to the others, which open it."""

    def __init__(self, device: int, handle: bytes | None = None):
        lib = load()
        h = _V()
        self.device = device
        if handle is None:
            st = lib.bs_bubble_sync_create(device, C.byref(h))
        else:
            buf = C.create_string_buffer(bytes(handle), 64)
            st = lib.bs_bubble_sync_open(device, buf, C.byref(h))
        if st != 0:
            raise BubbleSpecError(st, "bs_bubble_sync_create/open", "")
        self.handle = h

    def export(self) -> bytes:
        buf = C.create_string_buffer(64)
        st = load().bs_bubble_sync_export(self.handle, buf)
        if st != 0:
            raise BubbleSpecError(st, "bs_bubble_sync_export", "")
        return buf.raw

    def arrive(self, rank: int, rl_step: int, stream=None):
        st = load().bs_bubble_sync_arrive(self.handle, rank, rl_step, _stream(stream, self.device))
        if st != 0:
            raise BubbleSpecError(st, "bs_bubble_sync_arrive", "")

    def poll(self, world: int, rl_step: int, halt, stream=None):
        st = load().bs_bubble_sync_poll(self.handle, world, rl_step, _p(halt), _stream(stream, self.device))
        if st != 0:
            raise BubbleSpecError(st, "bs_bubble_sync_poll", "")

    def close(self):
        if self.handle:
            load().bs_bubble_sync_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def unified_attention_workspace_bytes(ctx_len, q_len, H_q: int, H_kv: int) -> int:
    """bs_unified_attention_workspace for host lists ctx_len / q_len."""
    import numpy as np

    ql = np.ascontiguousarray(np.asarray(q_len, dtype=np.int32))
    cl = np.ascontiguousarray(np.asarray(ctx_len, dtype=np.int32))
    ip = C.POINTER(C.c_int32)
    nbytes = C.c_int64()
    st = load().bs_unified_attention_workspace(len(ql), cl.ctypes.data_as(ip), ql.ctypes.data_as(ip), H_q, H_kv,
                                               C.byref(nbytes))
    if st != 0:
        raise BubbleSpecError(st, "bs_unified_attention_workspace", "")
    return int(nbytes.value)


def bs_unified_attention(q, k_cache, v_cache, page_table, ctx_len_dev, ctx_len, q_len, H_kv: int, out=None,
                         scale: float = 0.0, workspace=None, stream=None):
    """Unified variable-query-length decode attention (bs_unified_attention).  q [T, H_q, 128],
    k_cache / v_cache [num_pages, H_kv, 64, 128] (bf16 tensors, or int16 holding bf16 bits),
    page_table [B, max_pages] int32 and ctx_len_dev [B] int32 on the device; ctx_len / q_len the
    host copies (the launch plan).  Returns out [T, H_q, 128] (same dtype as q)."""
    import numpy as np

    lib = load()
    ql = np.ascontiguousarray(np.asarray(q_len, dtype=np.int32))
    cl = np.ascontiguousarray(np.asarray(ctx_len, dtype=np.int32))
    B = len(ql)
    H_q = q.shape[1]
    ip = C.POINTER(C.c_int32)
    if workspace is None:
        workspace = torch.empty(max(1, unified_attention_workspace_bytes(cl, ql, H_q, H_kv)), dtype=torch.uint8,
                                device=q.device)
    if out is None:
        out = torch.empty_like(q)
    st = lib.bs_unified_attention(_p(q), _p(k_cache), _p(v_cache), k_cache.shape[0], _p(page_table),
                                  page_table.shape[1], _p(ctx_len_dev), cl.ctypes.data_as(ip), ql.ctypes.data_as(ip),
                                  B, H_q, H_kv, q.shape[2], k_cache.shape[2], scale, _p(out), _p(workspace),
                                  workspace.numel(), _stream(stream, q.device.index))
    if st != 0:
        raise BubbleSpecError(st, "bs_unified_attention", "")
    return out


def bsx_synth_attn_values(out, base: int, mult: float, stream=None):
    st = load().bsx_synth_attn_values(_p(out), out.numel(), base & 0xFFFFFFFF, mult,
                                      _stream(stream, out.device.index))
    _chk(None, st, "bsx_synth_attn_values")


def bs_lm_head_logits(h, w, logits=None, row_key=None, row_bad=None, stream=None):
    """LM-head logits with fused row statistics (bs_lm_head_logits).  h [rows, d], w [V, d]
    (bf16, or int16 bf16 bits).  Returns (logits [rows, V] like h's dtype, row_key int64 [rows],
    row_bad int32 [rows])."""
    rows, d = h.shape
    V = w.shape[0]
    if logits is None:
        logits = torch.empty((rows, V), dtype=h.dtype, device=h.device)
    if row_key is None:
        row_key = torch.empty(rows, dtype=torch.int64, device=h.device)
    if row_bad is None:
        row_bad = torch.empty(rows, dtype=torch.int32, device=h.device)
    st = load().bs_lm_head_logits(_p(h), _p(w), rows, d, V, _p(logits), logits.stride(0), _p(row_key), _p(row_bad),
                                  _stream(stream, h.device.index))
    _chk(None, st, "bs_lm_head_logits")
    return logits, row_key, row_bad
