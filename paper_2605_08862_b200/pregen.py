"""Bubble pre-generation: a DP rank that finished its batch B_t
spends the inter-GPU bubble generating responses for the NEXT step's prompts, polling the
central synchronizer every T decoding steps (T = 50) and halting once every rank has
completed B_t.  Those partial responses become the next step's token pools
(P:197-200), routed to their owner ranks by bs_draft_exchange.

Everything on the device is a library call: plain decoding of the pre-generation slots
(RolloutEngine(plain=True): bsx_target_rows -> bs_verify_commit with draft_len = 0, i.e. Alg. 1
lines 4-7) and bs_bubble_sync_poll, captured together as one CUDA graph per chunk of T steps.
The host reads one pinned flag per chunk.  The pre-generation batch size is G samples per
prompt, the GRPO group size.
"""
from __future__ import annotations

import numpy as np
import torch

from .api import BubbleSync, Context
from .engine import RolloutEngine, Target


def pool_sequences(prompt_ids, prompt_tails, responses, lengths, M: int):
    """Pool sequences of the pre-generated responses (reading L4: [last M prompt tokens] +
    response; the prompt tail's -1 padding dropped; empty responses skipped).  Host arrays in,
    (seq_prompt int32, seq_off int64, tokens int32) out, in rollout order."""
    seqs, sp = [], []
    for b in range(len(prompt_ids)):
        L = int(lengths[b])
        if L <= 0:
            continue
        tail = [int(x) for x in prompt_tails[b][-M:] if x >= 0]
        seqs.append(np.asarray(tail + [int(x) for x in responses[b][:L]], dtype=np.int32))
        sp.append(int(prompt_ids[b]))
    off = np.zeros(len(seqs) + 1, dtype=np.int64)
    if seqs:
        off[1:] = np.cumsum([len(s) for s in seqs])
    tokens = np.concatenate(seqs) if seqs else np.zeros(0, dtype=np.int32)
    return np.asarray(sp, dtype=np.int32), off, tokens


class Pregenerator:
    """Pre-generation on rollout slots [slot0, slot0 + n) of `ctx` (spare slots beside the
    rank's own batch).  The ctx's bound response buffer (bs_rollout_bind_output) receives the
    generated tokens."""

    def __init__(self, ctx: Context, slot0: int, n: int, target: Target, sync: BubbleSync,
                 rank: int, world: int, temperature: float = 1.0, top_p: float = 1.0,
                 poll_every: int = 50, stream: torch.cuda.Stream | None = None):
        self.ctx, self.n, self.sync, self.rank, self.world = ctx, n, sync, rank, world
        self.poll_every = poll_every
        self.eng = RolloutEngine(ctx, n, 0, temperature, top_p, target, stream=stream, slot0=slot0,
                                 plain=True)
        self.stream = self.eng.stream
        dev = torch.device("cuda", ctx.device)
        self.halt = torch.zeros(1, dtype=torch.int32, device=dev)
        self.halt_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.graph = None
        self.graph_step = None
        self.rl_step = None
        self.steps = 0

    def begin(self, uids, prompt_ids, prompt_tail, max_len):
        """bs_rollout_begin of the next step's prompts (device tensors, n rows)."""
        self.eng.begin(uids, prompt_ids, prompt_tail, max_len)
        self.steps = 0

    def _capture(self, rl_step: int):
        """One chunk = poll_every plain decoding steps, then the synchronizer poll."""
        e = self.eng
        with torch.cuda.stream(self.stream):
            e.step()  # warm (attribute setup outside the capture); a real step
            self.sync.poll(self.world, rl_step, self.halt, stream=self.stream)
        self.stream.synchronize()
        self.steps += 1
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            for _ in range(self.poll_every):
                e.step()
            self.sync.poll(self.world, rl_step, self.halt, stream=self.stream)
        self.graph, self.graph_step = g, rl_step

    def run(self, rl_step: int, max_chunks: int | None = None) -> int:
        """Pre-generate until the synchronizer reports that all `world` ranks finished rl_step
        (or every pre-generation rollout reached its max length, or max_chunks).  Returns the
        decoding steps run."""
        if self.graph is None or self.graph_step != rl_step:
            self._capture(rl_step)
        chunks = 0
        with torch.cuda.stream(self.stream):
            while max_chunks is None or chunks < max_chunks:
                self.graph.replay()
                self.steps += self.poll_every
                chunks += 1
                self.halt_host.copy_(self.halt, non_blocking=True)
                self.stream.synchronize()
                if int(self.halt_host[0]) or self.eng.all_finished():
                    break
        return self.steps

    def pools(self, prompt_ids, prompt_tails, responses, M: int):
        """The pre-generated responses as pool sequences (host arrays; see pool_sequences)."""
        pos = torch.zeros(self.n, dtype=torch.int32, device=self.halt.device)
        self.ctx.bs_rollout_state(self.eng.slots, pos, None, stream=self.stream)
        self.stream.synchronize()
        return pool_sequences(prompt_ids, prompt_tails, responses, pos.cpu().numpy(), M)
