"""Multi-process (world size 2, gloo, CPU) coverage of the (b,h)-sharded path's host logic:
shard assignment, per-rank input generation equal to the single-process tensors, per-rank
oracle work on its own shard, max-over-ranks timing reduction and the verification gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_17245_b200.shard import batch_shard, max_over_ranks
from synth import CONFIGS, make_qkv


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    cfg = CONFIGS["C2"].with_(B=4, H=2, H_kv=2, N=97)
    b0, nb = batch_shard(cfg.B, rank, world)
    q, k, v = make_qkv(cfg, B=nb, head_offset=b0)
    # each rank computes the oracle on its own shard only (no data-path collective)
    out = oracle.attn_full(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                           block_l=cfg.block_l, G=cfg.group_size)
    t = max_over_ranks([1.0 + rank, 5.0 - rank])
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((b0, nb, out), gathered, dst=0)
    if rank == 0:
        ret["gathered"] = gathered
        ret["max"] = t
    dist.destroy_process_group()


def test_world2_sharded_matches_single_process():
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(worker, args=(world, free_port(), ret), nprocs=world, join=True)
    assert ret["max"] == [2.0, 5.0]
    cfg = CONFIGS["C2"].with_(B=4, H=2, H_kv=2, N=97)
    q, k, v = make_qkv(cfg)
    full = []
    for b0, nb, out in sorted(ret["gathered"], key=lambda x: x[0]):
        assert np.array_equal(out.shape, (nb, 2, 97, 64))
        full.append(out)
    full = np.concatenate(full)
    ref = __import__("oracle").attn_full(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                                         block_l=64, G=2)
    assert np.array_equal(full, ref)  # deterministic per head: bit-identical


def test_batch_shard_rules():
    assert batch_shard(32, 0, 8) == (0, 4) and batch_shard(32, 7, 8) == (28, 4)
    assert [batch_shard(32, r, 4) for r in range(4)] == [(0, 8), (8, 8), (16, 8), (24, 8)]
    with pytest.raises(ValueError):
        batch_shard(32, 0, 3)
    with pytest.raises(ValueError):
        batch_shard(32, 2, 2)
    assert max_over_ranks([1.5, 2]) == [1.5, 2.0]  # no process group: identity


# ---------------------------------------------------------------------------------------------
# Q-block (sequence) sharding: ranks split the 256-row Q tile pairs; K/V arrive sharded along N
# and are all_gathered once (the one exchange step); each rank computes only its Q rows.
from paper_2507_17245_b200.shard import (causal_work_of_shard, gather_kv_sequence_shards,  # noqa: E402
                                         q_pair_shard, q_rows_of_shard)


def seq_worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    cfg = CONFIGS["C4"].with_(B=1, H=1, H_kv=1, N=1000, d=64, causal=True)
    q, k, v = make_qkv(cfg)
    n_loc = cfg.N // world
    k_loc, v_loc = k[:, :, rank * n_loc:(rank + 1) * n_loc], v[:, :, rank * n_loc:(rank + 1) * n_loc]
    kf, vf = gather_kv_sequence_shards(k_loc, v_loc)
    assert torch.equal(kf, k) and torch.equal(vf, v)
    items = [(0, qb) for r0, r1 in q_rows_of_shard(cfg.N, rank, world, causal=True)
             for qb in range(r0 // cfg.block_l, -(-r1 // cfg.block_l))]
    out = oracle.attn_items(q.float().numpy(), kf.float().numpy(), vf.float().numpy(), items,
                            block_l=cfg.block_l, G=cfg.group_size, causal=True)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((items, out), gathered, dst=0)
    if rank == 0:
        ret["gathered"] = gathered
    dist.destroy_process_group()


def test_world2_q_block_sharding_matches_single_process():
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(seq_worker, args=(world, free_port(), ret), nprocs=world, join=True)
    cfg = CONFIGS["C4"].with_(B=1, H=1, H_kv=1, N=1000, d=64, causal=True)
    q, k, v = make_qkv(cfg)
    import oracle
    nqb = -(-cfg.N // cfg.block_l)
    ref = oracle.attn_items(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                            [(0, qb) for qb in range(nqb)], block_l=cfg.block_l, G=cfg.group_size,
                            causal=True)
    seen = set()
    for items, out in ret["gathered"]:
        for (bh, qb), o in zip(items, out):
            assert qb not in seen
            seen.add(qb)
            assert np.array_equal(o, ref[qb])  # deterministic per Q block: bit-identical
    assert seen == set(range(nqb))


def test_q_pair_shard_partition_and_causal_balance():
    for N in (1, 255, 256, 1000, 16384):
        for world in (1, 2, 3, 8):
            rows = sorted(r for rk in range(world) for r in q_rows_of_shard(N, rk, world))
            assert rows[0][0] == 0 and rows[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))  # disjoint, no gaps
    # zigzag slots over heaviest-first pairs: causal work within 3 % across 8 ranks at 16k
    w = [causal_work_of_shard(16384, rk, 8) for rk in range(8)]
    assert sum(w) == sum(qt + 1 for qt in range(128))
    assert max(w) / min(w) < 1.03, w
    assert q_pair_shard(3, 8) == (3, 8)
    with pytest.raises(ValueError):
        q_pair_shard(8, 8)


# ---------------------------------------------------------------------------------------------
# flattened (b, h) sharding for any B (no B % world requirement)
from paper_2507_17245_b200.shard import head_shard, make_head_shard  # noqa: E402


def test_head_shard_partition_any_batch():
    for B, H, Hkv in ((3, 4, 2), (1, 12, 12), (32, 32, 32), (4, 32, 8), (5, 2, 1)):
        for world in (1, 2, 3, 8):
            parts = [head_shard(B, H, Hkv, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == B * Hkv
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [u1 - u0 for u0, u1 in parts]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("u0,u1", [(0, 3), (1, 6), (5, 6), (2, 4)])
def test_make_head_shard_matches_full_tensors(u0, u1):
    cfg = CONFIGS["C3"].with_(B=3, H=4, H_kv=2, N=33, d=32)
    q, k, v = make_qkv(cfg)
    qs, ks, vs = make_head_shard(cfg, u0, u1)
    g = cfg.H // cfg.H_kv
    assert torch.equal(qs[0], q.reshape(-1, 33, 32)[u0 * g:u1 * g])
    assert torch.equal(ks[0], k.reshape(-1, 33, 32)[u0:u1])
    assert torch.equal(vs[0], v.reshape(-1, 33, 32)[u0:u1])


def head_worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    cfg = CONFIGS["C3"].with_(B=3, H=4, H_kv=2, N=70, d=32, block_l=64)  # B=3 over 2 ranks
    u0, u1 = head_shard(cfg.B, cfg.H, cfg.H_kv, rank, world)
    q, k, v = make_head_shard(cfg, u0, u1)
    out = oracle.attn_full(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                           block_l=cfg.block_l, G=cfg.group_size, causal=True)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((u0, u1, out), gathered, dst=0)
    if rank == 0:
        ret["gathered"] = gathered
    dist.destroy_process_group()


def test_world2_flattened_head_shards_match_single_process():
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(head_worker, args=(world, free_port(), ret), nprocs=world, join=True)
    cfg = CONFIGS["C3"].with_(B=3, H=4, H_kv=2, N=70, d=32, block_l=64)
    q, k, v = make_qkv(cfg)
    import oracle
    ref = oracle.attn_full(q.float().numpy(), k.float().numpy(), v.float().numpy(),
                           block_l=64, G=2, causal=True).reshape(-1, 70, 32)
    parts = sorted(ret["gathered"], key=lambda x: x[0])
    full = np.concatenate([o[0] for _, _, o in parts])
    assert np.array_equal(full, ref)
