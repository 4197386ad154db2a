"""RolloutEngine — drives Alg. 1's decoding loop on one GPU through the C-ABI.

One decoding step is four library calls and no host synchronisation:

    bs_draft_lookup -> bsx_target_rows (the synthetic target's "forward": which logits row
    is p_t for each position; a real engine runs its model here) -> bs_verify_step ->
    bs_commit

so a chunk of steps can be captured once into a CUDA graph and replayed.  The engine
owns the per-step device buffers; PyTorch only allocates them and provides the stream.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .api import Context


TARGET_MODES = {"position": 0, "markov": 1, "mixed": 2, "sample": 3}  # bsx_target_rows modes


@dataclass
class Target:
    """Synthetic target policy: logits rows live in `bank` [nbank, V] (bf16, on device) and
    the row for a position is workloads.target_row(spec, prompt, t, prev)."""
    bank: torch.Tensor
    nbank: int
    target_seed: int
    mode: int  # 0 position, 1 markov, 2 mixed, 3 sample (workloads.TargetSpec)


class RolloutEngine:
    def __init__(self, ctx: Context, n: int, k: int, temperature: float, top_p: float,
                 target: Target, stream: torch.cuda.Stream | None = None, fused: bool = True,
                 fuse_lookup: bool = True, top_k: int = 0, ngram: tuple | None = None,
                 slot0: int = 0, plain: bool = False):
        self.ctx, self.n, self.k = ctx, n, k
        self.fused = fused  # bs_verify_commit (one launch) instead of bs_verify_step + bs_commit
        # bs_verify_commit_lookup: each launch also looks up the next step's drafts (the first
        # step's lookup runs in begin()), so a decoding step is target rows + one launch
        # ngram = (n_min, n_max): drafts from the n-gram linear-scan drafter (bs_draft_lookup_ngram,
        # its own launch) instead of the suffix index
        self.ngram = ngram
        # plain = True: no drafts at all (draft_len stays 0): plain decoding, one sample per step
        # (Alg. 1 lines 4-7) -- the pre-generation of the next RL step's responses
        self.plain = plain
        self.fuse_lookup = fused and fuse_lookup and ngram is None and not plain
        self.launches_per_step = 2 if (self.fuse_lookup or plain) else 3
        self.T, self.top_p, self.top_k, self.target = temperature, top_p, top_k, target
        # the kernel right before each verify launch is bsx_target_rows (the synthetic model),
        # which writes only row_index: the verify may plan before its PDL wait
        ctx.bsx_set_early_plan(True)
        dev = torch.device("cuda", ctx.device)
        # a dedicated stream: CUDA graphs cannot be captured on the legacy default stream
        self.stream = stream or torch.cuda.Stream(dev)
        i32 = dict(dtype=torch.int32, device=dev)
        self.slots = torch.arange(slot0, slot0 + n, **i32)  # this engine's rollout slots
        self.draft = torch.full((n, max(k, 1)), -1, **i32)
        self.draft_len = torch.zeros(n, **i32)
        self.match_len = torch.zeros(n, **i32)
        self.row_index = torch.zeros((n, k + 1), dtype=torch.int64, device=dev)
        self.out_tokens = torch.full((n, k + 1), -1, **i32)
        self.out_len = torch.zeros(n, **i32)
        self.out_acc = torch.zeros(n, **i32)
        self.finished = torch.zeros(n, **i32)
        self.live = torch.zeros(1, **i32)  # bs_rollout_live output
        self.rl_step = 0
        self.graph = None
        self.graph_steps = 0

    # ------------------------------------------------------------------ RL-step setup
    def put_pools(self, rl_step, seq_prompt, seq_off, tokens):
        """bs_draft_pool_put of device tensors (int32 prompt ids, int64 offsets, int32 tokens)."""
        n_tok = int(tokens.numel())
        self._sync_inputs()
        self.ctx.bs_draft_pool_put(rl_step, seq_prompt, seq_off, tokens, n_tok, stream=self.stream)

    def seal(self, rl_step):
        self.ctx.bs_draft_pool_seal(rl_step, stream=self.stream)
        self.rl_step = rl_step

    def _sync_inputs(self):
        """Order the engine stream after work the caller queued on its current stream."""
        cur = torch.cuda.current_stream(self.stream.device)
        if cur != self.stream:
            self.stream.wait_stream(cur)

    def begin(self, uids, prompt_ids, prompt_tail, max_len):
        self._sync_inputs()
        self.ctx.bs_rollout_begin(self.slots, uids, prompt_ids, prompt_tail, max_len,
                                  stream=self.stream)
        if self.fuse_lookup:  # the first step's drafts (later ones come from the verify launch)
            self.ctx.bs_draft_lookup(self.rl_step, self.slots, self.k, self.draft, self.draft_len,
                                     self.match_len, stream=self.stream)

    # ------------------------------------------------------------------ decoding
    def _lookup(self):
        c, k, s = self.ctx, self.k, self.stream
        if self.ngram is not None:
            c.bs_draft_lookup_ngram(self.rl_step, self.slots, k, self.ngram[0], self.ngram[1], self.draft,
                                    self.draft_len, self.match_len, stream=s)
        else:
            c.bs_draft_lookup(self.rl_step, self.slots, k, self.draft, self.draft_len, self.match_len,
                              stream=s)

    def step(self):
        c, k, s = self.ctx, self.k, self.stream
        if not self.fuse_lookup and not self.plain:
            self._lookup()
        t = self.target
        c.bsx_target_rows(self.slots, self.draft, self.draft_len, k, t.target_seed, t.mode,
                          t.nbank, self.row_index, stream=s)
        if self.fuse_lookup:
            c.bs_verify_commit_lookup(self.rl_step, self.slots, t.bank, self.row_index, t.bank.shape[1],
                                      self.draft, self.draft_len, k, self.T, self.top_p, self.out_tokens,
                                      self.out_len, self.out_acc, self.finished, self.match_len, stream=s,
                                      top_k=self.top_k)
        elif self.fused:
            c.bs_verify_commit(self.slots, t.bank, self.row_index, t.bank.shape[1], self.draft,
                               self.draft_len, k, self.T, self.top_p, self.out_tokens, self.out_len,
                               self.out_acc, self.finished, stream=s, top_k=self.top_k)
        else:
            c.bs_verify_step(self.slots, t.bank, self.row_index, t.bank.shape[1], self.draft,
                             self.draft_len, k, self.T, self.top_p, self.out_tokens, self.out_len,
                             self.out_acc, stream=s, top_k=self.top_k)
            c.bs_commit(self.slots, self.out_tokens, self.out_len, k, self.finished, stream=s)

    # target rows + verify (fused commit and next lookup), or lookup + target rows + verify;
    # top-p < 1 adds the plan / commit / lookup kernels

    def capture(self, steps: int):
        """Capture `steps` decoding steps into one CUDA graph (replayed by run_graph)."""
        with torch.cuda.stream(self.stream):
            self.step()  # warm (first-call attribute setup happens outside the capture)
        self.stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            for _ in range(steps):
                self.step()
        self.graph, self.graph_steps = g, steps
        return g

    def run_graph(self):
        with torch.cuda.stream(self.stream):
            self.graph.replay()

    def live_count(self):
        """Enqueue bs_rollout_live on the engine stream; returns the device int32 [1] holding the
        number of this engine's rollouts not yet finished."""
        self.ctx.bs_rollout_live(self.slots, self.live, stream=self.stream)
        return self.live

    def all_finished(self) -> bool:
        with torch.cuda.stream(self.stream):
            live = self.live_count()
            self.stream.synchronize()
            return int(live.item()) == 0

    def run_until_done(self, max_steps: int = 1 << 20, chunk: int = 64, use_graph: bool = True):
        """Decode until every rollout finished (EOS or max_len); host checks once per chunk."""
        steps = 0
        if use_graph and (self.graph is None or self.graph_steps != chunk):
            self.capture(chunk)
            steps = 1  # capture() ran one real (eager) warm-up step
        while steps < max_steps:
            if use_graph:
                self.run_graph()
                steps += chunk
            else:
                for _ in range(chunk):
                    self.step()
                steps += chunk
            if self.all_finished():
                break
        return steps

    def stats(self, reset: bool = False):
        st = self.ctx.bs_stats_read(reset=reset, stream=self.stream)
        return summarize_stats(st)


def summarize_stats(st: np.ndarray) -> dict:
    """AL / DL / AR and streak histogram from the device counters (
    identity AR = (AL - 1) / DL pinned by P:269)."""
    st = st.astype(np.int64)
    spec, plain = int(st[0]), int(st[1])
    emit_spec, emit_plain = int(st[2]), int(st[3])
    acc, prop = int(st[4]), int(st[5])
    out = {
        "verify_steps": spec, "plain_steps": plain, "decode_steps": spec + plain,
        "tokens": emit_spec + emit_plain, "accepted": acc, "proposed": prop,
        "rows_verified": int(st[6]), "rows_needed": int(st[7]),
        "acceptance_length": emit_spec / spec if spec else None,
        "draft_length": prop / spec if spec else None,
        "acceptance_rate": acc / prop if prop else None,
        "streak_hist": [int(x) for x in st[8:41]],
    }
    return out
