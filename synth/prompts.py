"""Seeded synthetic prompts and forced-acceptance corruption draws.

Prompts: i.i.d. uniform token ids in [0, V) from seed 1, drawn for the GLOBAL
batch so a data-parallel shard sees the same rows as a 1-GPU run.
Corruption slots (forced-acceptance benchmarking): slot j in 1..k with
P(j) = alpha^(j-1) (1 - alpha), and k+1 (= no corruption) with P = alpha^k, drawn per
(step, global sequence) from seed 2. Only random draws live here.
"""
from __future__ import annotations

import numpy as np
import torch


def make_prompts(batch: int, prompt_len: int, vocab: int, seed: int = 1) -> torch.Tensor:
    g = torch.Generator().manual_seed(seed)
    return torch.randint(0, vocab, (batch, prompt_len), generator=g, dtype=torch.int64).to(torch.int32)


def make_corrupt_slots(steps: int, batch: int, k: int, alpha: float, seed: int = 2) -> np.ndarray:
    """[steps, batch] int32 in 1..k+1 (k+1 means: draft left intact)."""
    rng = np.random.default_rng(seed)
    u = rng.random((steps, batch))
    probs = np.array([alpha ** (j - 1) * (1 - alpha) for j in range(1, k + 1)] + [alpha ** k])
    cdf = np.cumsum(probs)
    cdf[-1] = 1.0
    return (np.searchsorted(cdf, u, side="right") + 1).astype(np.int32)
