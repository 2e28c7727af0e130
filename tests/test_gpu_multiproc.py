"""Multi-process runs of the CUDA library (world size 2 on ONE GPU, gloo for the host-side
gather): each rank computes its shard through the C-ABI — flattened (b, h) units for any B, or
Q tile pairs — and rank 0 gathers the outputs; they must be bit-identical to one single-process
call over the whole job (every (b, h) problem and every Q tile pair is independent, §3.3 P:304,
and each is computed by the same kernel code). This is the verification step of the north
star's 8-GPU layout ("NCCL is used only to gather results for verification") run with gloo so it
fits the one-GPU box."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_17245_b200.shard import head_shard, make_head_shard, q_pair_shard, q_rows_of_shard
from synth import CONFIGS, make_qkv

pytestmark = pytest.mark.gpu
CFG = CONFIGS["C3"].with_(B=3, H=8, H_kv=2, N=700, d=64, block_l=128)  # B=3 over 2 ranks, GQA


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, mode, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2507_17245_b200 as da
    if mode == "heads":
        u0, u1 = head_shard(CFG.B, CFG.H, CFG.H_kv, rank, world)
        q, k, v = make_head_shard(CFG, u0, u1, device="cuda")
        out = da.distr_attn_fwd_ex(q, k, v, block_l=CFG.block_l, group_size=2, seed=4, causal=True)
        payload = (u0, u1, out.cpu())
    else:  # Q tile pairs of every head
        q, k, v = make_qkv(CFG, device="cuda")
        out = torch.zeros_like(q)
        da.distr_attn_fwd_ex(q, k, v, out, block_l=CFG.block_l, group_size=2, seed=4, causal=True,
                             q_shard=q_pair_shard(rank, world))
        payload = (q_rows_of_shard(CFG.N, rank, world, causal=True), out.cpu())
    torch.cuda.synchronize()
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(payload, gathered, dst=0)
    if rank == 0:
        ret["gathered"] = gathered
    dist.destroy_process_group()


def single_process():
    import paper_2507_17245_b200 as da
    q, k, v = make_qkv(CFG, device="cuda")
    out = da.distr_attn_fwd_ex(q, k, v, block_l=CFG.block_l, group_size=2, seed=4, causal=True)
    torch.cuda.synchronize()
    return out.cpu()


@pytest.mark.parametrize("mode", ["heads", "qpairs"])
def test_world2_cuda_shards_bit_identical_to_single_process(mode):
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(worker, args=(world, free_port(), mode, ret), nprocs=world, join=True)
    ref = single_process()
    g = CFG.H // CFG.H_kv
    if mode == "heads":
        flat = ref.reshape(-1, CFG.N, CFG.d)
        covered = 0
        for u0, u1, out in ret["gathered"]:
            assert torch.equal(out[0], flat[u0 * g:u1 * g])
            covered += u1 - u0
        assert covered == CFG.B * CFG.H_kv
    else:
        seen = 0
        for rows, out in ret["gathered"]:
            for r0, r1 in rows:
                assert torch.equal(out[:, :, r0:r1], ref[:, :, r0:r1])
                seen += r1 - r0
        assert seen == CFG.N
