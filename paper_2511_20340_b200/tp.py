"""Tensor parallelism plumbing around the C ABI: one process per GPU (torchrun), all
ranks serve the same global batch; rank r's handle is built with tp_size = world, tp_rank = r and
holds its weight slices (engine.pack_weights), and the ranks' handles join one NCCL communicator
whose all-reduces run inside the library's decode step (graph-captured). torch.distributed only
carries the 128-byte NCCL unique id from rank 0 to the others.
"""
from __future__ import annotations

from collections.abc import Mapping

import torch.distributed as dist


def share_unique_id(make_id, rank: int) -> bytes:
    """Rank 0 calls make_id() (e.g. engine.nccl_unique_id); every rank returns its bytes."""
    obj = [make_id() if rank == 0 else None]
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast_object_list(obj, src=0)
    return obj[0]


def share_xch_handles(own: bytes, rank: int, world: int) -> list[bytes]:
    """NEXT-3: all-gather every rank's 64-byte exchange-region handle (Engine.xch_handle), in rank
    order, for Engine.attach_xch. Only the host carries the handles; the data path never touches
    torch.distributed."""
    if len(own) != 64:
        raise ValueError("an exchange handle is 64 bytes")
    if world == 1:
        return [own]
    out = [None] * world
    dist.all_gather_object(out, (rank, own))
    got = dict(out)
    if sorted(got) != list(range(world)):
        raise RuntimeError(f"exchange handles from ranks {sorted(got)}, expected 0..{world - 1}")
    return [got[q] for q in range(world)]


class LazyWeights(Mapping):
    """A weight dict whose tensors are drawn on access (synth.make_weights with names={name}), so a
    rank never holds more than one full tensor besides its packed slices (70B: 141 GB of bf16)."""

    def __init__(self, make_one, names):
        self._make_one = make_one
        self._names = list(names)

    def __getitem__(self, name):
        if name not in self._names:
            raise KeyError(name)
        return self._make_one(name)

    def __iter__(self):
        return iter(self._names)

    def __len__(self):
        return len(self._names)
