"""Multi-GPU plumbing: partition independent tracking units over ranks and
gather their epoch records once at the end.

The path has no per-epoch exchange -- channels never share mutable state
(pipeline.hpp:88-90) -- so ranks run independently and the
only collective is the end-of-run gather of records to rank 0 (NCCL over
NVLink on GPUs, gloo in the CPU tests).

Units per config: recordings (config 4, strong), channel batches of one
stream broadcast from rank 0 (configs 2/3, strong), PRNs of one recording
(config 5, strong; the planes are gathered).  Config 1 (a single sequential
channel) does not shard: N ranks run N replicas.
"""
from __future__ import annotations

from typing import List, Sequence


def shard_range(n_units: int, world: int, rank: int) -> range:
    """Contiguous, balanced slice of n_units for `rank` (sizes differ by at
    most one; every unit is owned by exactly one rank)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def shard_list(units: Sequence, world: int, rank: int) -> List:
    return [units[i] for i in shard_range(len(units), world, rank)]


def broadcast_stream(buf, dist, src: int = 0):
    """Broadcasts a recording (1-D uint8 tensor, same size on every rank)
    from `src` to every rank: the stream that all channel batches of a run
    share (configs 2/3).  NCCL over NVLink on GPUs, gloo in the CPU tests."""
    if dist is not None and dist.get_world_size() > 1:
        dist.broadcast(buf, src=src)
    return buf


def gather_bytes(local, dist, dst: int = 0):
    """Gathers a 1-D uint8 torch tensor of per-rank records to `dst` (sizes may
    differ: they are exchanged first).  Returns the list of tensors on dst,
    None elsewhere.  Works for NCCL (CUDA tensors) and gloo (CPU tensors)."""
    import torch
    world = dist.get_world_size()
    rank = dist.get_rank()
    size = torch.tensor([local.numel()], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(size) for _ in range(world)]
    dist.all_gather(sizes, size)
    n_max = int(max(int(s.item()) for s in sizes))
    buf = torch.zeros(n_max, dtype=torch.uint8, device=local.device)
    buf[: local.numel()] = local
    if dist.get_backend() == "gloo":
        outs = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(outs, buf)  # gloo has no gather for all dtypes
        if rank != dst:
            return None
    else:
        outs = [torch.zeros_like(buf) for _ in range(world)] if rank == dst else None
        dist.gather(buf, outs, dst=dst)
        if rank != dst:
            return None
    return [o[: int(s.item())] for o, s in zip(outs, sizes)]
