"""Sharding of independent fronts across GPUs (BASELINE config 3).

One process per GPU.  Fronts of a multifrontal level are independent, so each
rank factors and solves its own contiguous shard with the batched kernels and
there is no collective on the data path.  The only communication is the
max-over-ranks time reduction of the benchmark and one gather of per-front
scalars (ranks, iteration counts) at the end.  Works with any
torch.distributed backend (NCCL on the B200 box, gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np


def shard_range(rank: int, world: int, per_rank: int) -> range:
    """Global front indices (= generator seeds) owned by ``rank``."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return range(rank * per_rank, (rank + 1) * per_rank)


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (the timed region's milliseconds)."""
    import torch
    dist = _dist()
    if dist is None:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_front_scalars(local, device=None) -> np.ndarray:
    """Concatenate per-front scalar rows from every rank in rank order."""
    import torch
    local = np.asarray(local)
    dist = _dist()
    if dist is None:
        return local.copy()
    t = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float64))
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return np.concatenate([p.cpu().numpy() for p in parts]).astype(local.dtype)
