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
