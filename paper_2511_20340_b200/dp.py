"""Data parallelism over the request batch: one process per GPU, each rank owns a
contiguous slice of the global batch and a full replica of the weights; sequences are independent,
so the hot path has NO collective. torch.distributed is used only around the timed region: a
barrier on both sides, the max of the ranks' device times and the sum of their token counts.
Backend-agnostic (nccl on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world():
    """(rank, world_size, local_rank) from the torchrun environment (1 process when absent)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_rows(global_rows: torch.Tensor, rank: int, world_size: int) -> torch.Tensor:
    """Rank r gets rows [r B, (r+1) B) of a [world_size * B, ...] tensor (weak scaling: B fixed per rank)."""
    n = global_rows.shape[0]
    if n % world_size:
        raise ValueError(f"global batch {n} not divisible by world size {world_size}")
    b = n // world_size
    return global_rows[rank * b:(rank + 1) * b].contiguous()


def reduce_timing(ms: float, tokens: float, device="cpu"):
    """(max over ranks of the timed-region milliseconds, sum over ranks of tokens)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return ms, tokens
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    n = torch.tensor([tokens], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return float(t.item()), float(n.item())


def gather_rows(local: torch.Tensor, device="cpu") -> torch.Tensor:
    """All ranks' equal-shaped slices concatenated in rank order (result checking only)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    parts = [torch.empty_like(local, device=device) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, local.to(device))
    return torch.cat(parts, 0)
