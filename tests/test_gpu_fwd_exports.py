"""GPU parity of the path that runs: the LSH exports of the FORWARD call itself.

For bf16 inputs the forward hashes every Q block inside the attention CTA (attn.cu
qhat_prologue); distr_attn_hash runs a different kernel (prep.cu hash_cta). The north star asks
for bit-exact bucket ids on all five configs (§3.2, Fig. 5), so these tests call
distr_attn_fwd_ex with the bucket_ids / perm exports and compare them, bit for bit, with
oracle.hash_all — on the five BASELINE configs at their own shapes (C5 at full B=32), on every
C4 sweep point the sweep reports (N = 4k..64k x G* in {2, 4} x block_l in {128, 256}), and on
stress inputs (U(0,1) ties, column clusters, zero columns, power-of-two scaling, the ragged
5-row block of N=197, GQA + causal). Outputs are compared with the oracle on sampled Q blocks
(each block is an independent unit of the method, §3.3) within max-abs 2e-2 / mean-abs 2e-3.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2507_17245_b200 as da
from gpu_util import MAX_ABS, MEAN_ABS, errors, gather_items, oracle_items, to_np32, valid_rows_mask
from synth import C4_SWEEP_N, CONFIGS, Config, make_qkv, sample_items

pytestmark = pytest.mark.gpu
DEV = "cuda"


def fwd_with_exports(q, k, v, cfg: Config, seed: int, G=None):
    B, H, N, d = q.shape
    nqb = -(-N // cfg.block_l)
    bk = torch.full((B, H, nqb, d), -1, dtype=torch.int16, device=DEV)
    pm = torch.full((B, H, nqb, d), 255, dtype=torch.uint8, device=DEV)
    out = da.distr_attn_fwd_ex(q, k, v, block_l=cfg.block_l, group_size=cfg.group_size if G is None else G,
                               seed=seed, causal=cfg.causal, bucket_ids=bk, perm=pm)
    torch.cuda.synchronize()
    return out, bk.cpu().numpy().view(np.uint16), pm.cpu().numpy()


def assert_exports_match(q, bk, pm, block_l, seed, heads=None):
    """Bit-exact comparison of the forward's exports with the oracle, per (b, h)."""
    B, H = q.shape[:2]
    heads = heads if heads is not None else [(b, h) for b in range(B) for h in range(H)]
    # one oracle call over the selected heads (stacked as a [1, n, N, d] tensor)
    qs = torch.stack([q[b, h] for b, h in heads]).unsqueeze(0)
    ob, op = oracle.hash_all(to_np32(qs), block_l, seed)
    for i, (b, h) in enumerate(heads):
        bad = np.argwhere(bk[b, h] != ob[0, i])
        assert bad.size == 0, ("bucket ids differ", b, h, bad[:5].tolist())
        assert np.array_equal(pm[b, h], op[0, i]), ("perm differs", b, h)


def assert_output_parity(q, k, v, out, cfg, items, seed, G=None):
    G = cfg.group_size if G is None else G
    want = oracle_items(q, k, v, items, block_l=cfg.block_l, G=G, seed=seed, causal=cfg.causal)
    got = gather_items(out, items, cfg.block_l)
    mask = valid_rows_mask(items, cfg.N, cfg.block_l, cfg.d)
    assert np.isfinite(got[mask]).all()
    mx, mean = errors(got, want, mask)
    assert mx <= MAX_ABS and mean <= MEAN_ABS, (cfg.name, mx, mean)
    return mx, mean


# ------------------------------------------------------------------------------ the five configs
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_forward_exports_all_configs(name):
    cfg = CONFIGS[name]
    q, k, v = make_qkv(cfg, device=DEV)
    out, bk, pm = fwd_with_exports(q, k, v, cfg, seed=0)
    if name == "C5":  # 1024 heads: first, last and a spread of others (all 128 blocks of each)
        heads = [(0, 0), (31, 31), (7, 3), (16, 17), (25, 30), (3, 28)]
        items = sample_items(cfg, n_heads=4, per_head=3)
    else:
        heads = None
        items = (None if cfg.B * cfg.H * cfg.nqb <= 2048 else sample_items(cfg, n_heads=4, per_head=4))
    assert_exports_match(q, bk, pm, cfg.block_l, 0, heads)
    if items is None:
        items = [(bh, qb) for bh in range(cfg.B * cfg.H) for qb in range(cfg.nqb)]
    assert_output_parity(q, k, v, out, cfg, items, seed=0)


# ------------------------------------------------------------------------------ C4 sweep points
@pytest.mark.parametrize("N", C4_SWEEP_N)
@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("block_l", [128, 256])
def test_forward_exports_c4_sweep_points(N, G, block_l):
    cfg = CONFIGS["C4"].with_(N=N, group_size=G, block_l=block_l)
    q, k, v = make_qkv(cfg, device=DEV)
    out, bk, pm = fwd_with_exports(q, k, v, cfg, seed=0)
    assert_exports_match(q, bk, pm, block_l, 0)  # all 16 heads, every block
    items = sample_items(cfg, n_heads=2, per_head=2 if N >= 32768 else 3)
    assert_output_parity(q, k, v, out, cfg, items, seed=0)


# ------------------------------------------------------------------------------ stress inputs
def _cfg(**kw):
    base = dict(name="s", B=1, H=4, N=197, d=64, block_l=64, group_size=2, causal=False,
                dtype="bf16", data_seed=21)
    base.update(kw)
    base.setdefault("H_kv", base["H"])
    return Config(**base)


# shapes of the configs the kernel instantiates: C2's ragged N=197 at l=64, C3's GQA + causal
# l=128, d=128 at l=128 and 256, d=32
STRESS_SHAPES = [
    dict(N=197, d=64, block_l=64, H=6),
    dict(N=1100, d=64, block_l=128, H=4, H_kv=1, causal=True),
    dict(N=1300, d=128, block_l=128, H=2),
    dict(N=700, d=128, block_l=256, H=2, group_size=4),
    dict(N=300, d=128, block_l=64, H=2),
    dict(N=333, d=32, block_l=128, H=3),
]


@pytest.mark.parametrize("shape", range(len(STRESS_SHAPES)))
@pytest.mark.parametrize("dist", ["uniform", "clustered", "zero_pow2"])
def test_forward_exports_stress(shape, dist):
    cfg = _cfg(**STRESS_SHAPES[shape])
    if dist == "zero_pow2":
        q, k, v = make_qkv(cfg, device=DEV)
        zc = [0, 5, cfg.d - 1]
        q[..., zc] = 0
        q = q.contiguous()
        out, bk, pm = fwd_with_exports(q, k, v, cfg, seed=9)
        assert_exports_match(q, bk, pm, cfg.block_l, 9)
        assert np.all(bk[..., zc] == 0)  # zero column -> all bits 0 -> bucket 0 (R5)
        # scaling Q by 2^-7 scales every fma-chain term exactly: identical bucket ids
        q2 = (q * 2.0 ** -7).contiguous()
        _, bk2, pm2 = fwd_with_exports(q2, k, v, cfg, seed=9)
        assert np.array_equal(bk, bk2) and np.array_equal(pm, pm2)
    else:
        q, k, v = make_qkv(cfg, dist=dist, device=DEV)
        out, bk, pm = fwd_with_exports(q, k, v, cfg, seed=9)
        assert_exports_match(q, bk, pm, cfg.block_l, 9)
        if dist == "uniform":  # the tie-heavy case (~43 tied buckets per 128)
            ties = sum(int(len(bk[0, h, b]) - len(np.unique(bk[0, h, b])))
                       for h in range(cfg.H) for b in range(cfg.nqb))
            assert ties > 0
    items = [(bh, qb) for bh in range(cfg.B * cfg.H) for qb in range(cfg.nqb)]
    assert_output_parity(q, k, v, out, cfg, items, seed=9)
