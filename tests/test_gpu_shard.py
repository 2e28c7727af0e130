"""Q-block (sequence) sharding on the GPU: the shards of a
world computed one after another into one output buffer reproduce the unsharded call bit for bit
(the per-tile arithmetic does not depend on the shard), and each shard writes only its own rows
(shard.q_rows_of_shard)."""
import pytest
import torch

import paper_2507_17245_b200 as da
from paper_2507_17245_b200.shard import q_pair_shard, q_rows_of_shard
from synth import CONFIGS, make_qkv

pytestmark = pytest.mark.gpu


def fwd(kind, q, k, v, out, causal, shard=None):
    if kind == "distr":
        return da.distr_attn_fwd_ex(q, k, v, out, block_l=128, group_size=2, causal=causal, q_shard=shard)
    if kind == "exact":
        return da.exact_attn_fwd_ex(q, k, v, out, causal=causal, q_shard=shard)
    return da.distr_attn_global_fwd_ex(q, k, v, out, group_size=2, causal=causal, q_shard=shard)


@pytest.mark.parametrize("kind", ["distr", "exact", "global"])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_equals_unsharded(kind, causal, world):
    cfg = CONFIGS["C4"].with_(B=1, H=2, H_kv=2, N=1500, causal=causal)
    q, k, v = make_qkv(cfg, device="cuda")
    full = fwd(kind, q, k, v, torch.empty_like(q), causal)
    sentinel = torch.full_like(q, float("nan"))
    for rank in range(world):
        part = fwd(kind, q, k, v, sentinel.clone(), causal, q_pair_shard(rank, world))
        rows = torch.zeros(cfg.N, dtype=torch.bool, device="cuda")
        for r0, r1 in q_rows_of_shard(cfg.N, rank, world, causal):
            rows[r0:r1] = True
        assert torch.equal(part[:, :, rows], full[:, :, rows]), (rank, kind)
        assert torch.isnan(part[:, :, ~rows]).all(), "wrote rows outside its shard"
