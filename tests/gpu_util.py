"""Helpers for the GPU parity tests: build the same seeded inputs for the CUDA path (device
tensors) and the oracle (numpy)."""
from __future__ import annotations

import numpy as np

from workloads import TargetSpec, bank_rows, make_pools, prompt_tails


def to_dev(a, dtype=None):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def bank_numpy(spec: TargetSpec) -> np.ndarray:
    return bank_rows(spec.bank_seed, np.arange(spec.nbank), spec.V, spec.beta)


def setup_rollouts(spec: TargetSpec, n_prompts: int, G_roll: int, M: int, max_len, seed=7):
    """Prompt tails and per-rollout metadata: rollouts b = p*G_roll + g."""
    prompts = np.arange(n_prompts, dtype=np.int32) * 3 + 1
    tails = prompt_tails(seed, prompts, M, spec.V)
    n = n_prompts * G_roll
    pid = np.repeat(prompts, G_roll).astype(np.int32)
    tail_rows = np.repeat(tails, G_roll, axis=0).astype(np.int32)
    uids = (np.arange(n, dtype=np.uint64) + np.uint64(1000003) * np.uint64(seed))
    ml = np.broadcast_to(np.asarray(max_len, dtype=np.int32), (n,)).copy()
    return prompts, tails, pid, tail_rows, uids, ml


def pools_for(spec: TargetSpec, prompts, tails, G: int, lens, match_rate: float, prefix: int,
              noise: float = 0.02):
    lens = np.asarray(lens).reshape(len(prompts), G)
    return make_pools(spec, prompts, tails, G, lens, match_rate, noise=noise, prefix=prefix)
