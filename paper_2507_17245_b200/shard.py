"""(b, h) sharding of the DistrAttention job across ranks.

Every (b, h) problem is independent (§3.3), so ranks split the batch into contiguous
slices and run the whole hot path on their slice with no collective in the data path. Only the
bench's timing reduction (max over ranks) and verification gathers use torch.distributed, and
always outside the timed region.
"""
from __future__ import annotations


def batch_shard(B: int, rank: int, world: int) -> tuple[int, int]:
    """(first batch index, batch count) of `rank`'s contiguous slice; B must divide evenly."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if B % world:
        raise ValueError(f"B={B} is not divisible by world size {world}")
    per = B // world
    return rank * per, per


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity without a process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(x) for x in values]
    t = torch.tensor([float(x) for x in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()
