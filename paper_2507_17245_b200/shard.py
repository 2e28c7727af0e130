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


def head_shard(B: int, H: int, H_kv: int, rank: int, world: int) -> tuple[int, int]:
    """[u0, u1) of the flattened KV units u = b*H_kv + h_kv `rank` owns (each unit carries its
    H/H_kv query heads, flattened q heads [u0*g, u1*g) with g = H/H_kv): contiguous, sizes differ
    by at most one, any B (no divisibility requirement; SURVEY §8(e) "(batch, head)")."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if H % H_kv:
        raise ValueError("H must be a multiple of H_kv")
    U = B * H_kv
    base, extra = divmod(U, world)
    u0 = rank * base + min(rank, extra)
    return u0, u0 + base + (1 if rank < extra else 0)


def make_head_shard(cfg, u0: int, u1: int, *, device="cpu", dist: str = "normal"):
    """Inputs of KV units [u0, u1) as one flattened batch: q [1, (u1-u0)*g, N, d], k/v
    [1, u1-u0, N, d] — exactly the rows the full single-process tensors hold for those heads
    (synth.make_qkv draws per batch element, so the covering batch elements are drawn and
    sliced)."""
    import torch
    from synth import make_qkv
    g = cfg.H // cfg.H_kv
    b0, b1 = u0 // cfg.H_kv, -(-u1 // cfg.H_kv)
    q, k, v = make_qkv(cfg, B=b1 - b0, head_offset=b0, device=device, dist=dist)
    lo = u0 - b0 * cfg.H_kv
    n = u1 - u0
    qf = q.reshape(1, -1, cfg.N, cfg.d)[:, lo * g:(lo + n) * g]
    kf = k.reshape(1, -1, cfg.N, cfg.d)[:, lo:lo + n]
    vf = v.reshape(1, -1, cfg.N, cfg.d)[:, lo:lo + n]
    return qf.contiguous(), kf.contiguous(), vf.contiguous()


def max_over_ranks(values, device=None):
    """Element-wise max of a list of floats over all ranks (identity without a process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(x) for x in values]
    t = torch.tensor([float(x) for x in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


# ---------------------------------------------------------------------------------------------
# Q-block (sequence) sharding — SURVEY §8(e) NEXT / §8(f) row 3: when B·H is smaller than the
# number of GPUs (long single-head runs), ranks split the 256-row Q tile pairs of every head
# instead of the heads. Every rank needs all of K and V (one all_gather if they arrive sharded
# along N); the attention itself has no collective. Slots are dealt in a zigzag (round x: rank
# takes slot x*world + rank for even x, x*world + world-1-rank for odd x); the kernel visits
# slots heaviest-first when causal, so every rank gets a near-equal share of the causal work.

TILE_PAIR_ROWS = 256


def q_pair_shard(rank: int, world: int) -> tuple[int, int]:
    """(offset, stride) for da_params.q_shard_offset / q_shard_stride."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return rank, world


def q_rows_of_shard(N: int, rank: int, world: int, causal: bool = False) -> list[tuple[int, int]]:
    """Row ranges [r0, r1) of Q whose outputs `rank` computes (mirrors the kernel's slot -> tile
    pair mapping: pair = slot, or npairs - 1 - slot when causal)."""
    npairs = -(-N // TILE_PAIR_ROWS)
    off, stride = q_pair_shard(rank, world)
    rows = []
    for x in range(-(-npairs // stride)):
        slot = x * stride + (stride - 1 - off if x & 1 else off)
        if slot >= npairs:
            continue
        pair = npairs - 1 - slot if causal else slot
        rows.append((pair * TILE_PAIR_ROWS, min(N, (pair + 1) * TILE_PAIR_ROWS)))
    return sorted(rows)


def causal_work_of_shard(N: int, rank: int, world: int) -> int:
    """Number of (query tile, key tile) 128x128 steps `rank` runs for a causal problem."""
    work = 0
    for r0, r1 in q_rows_of_shard(N, rank, world, causal=True):
        for qt in range(r0 // 128, -(-r1 // 128)):
            work += qt + 1
    return work


def gather_kv_sequence_shards(k_local, v_local, group=None):
    """all_gather K/V shards split along N (dim 2) -> full K, V on every rank (the one exchange
    step of Q-block sharding; outside the attention kernel)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    ks = [torch.empty_like(k_local) for _ in range(world)]
    vs = [torch.empty_like(v_local) for _ in range(world)]
    dist.all_gather(ks, k_local.contiguous(), group=group)
    dist.all_gather(vs, v_local.contiguous(), group=group)
    return torch.cat(ks, dim=2).contiguous(), torch.cat(vs, dim=2).contiguous()
