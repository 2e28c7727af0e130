"""Helpers shared by the GPU parity tests (tolerances, oracle calls on sampled items)."""
import numpy as np
import torch

import oracle

# north_star: outputs within max-abs 2e-2 and mean-abs 2e-3 of the oracle for bf16 inputs with
# fp32 accumulation.
MAX_ABS = 2e-2
MEAN_ABS = 2e-3


def to_np32(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy()


def gather_items(out: torch.Tensor, items, block_l: int) -> np.ndarray:
    """GPU output rows for work items (bh, qb) -> [n, block_l, d] float64 (rows past N = 0)."""
    B, H, N, d = out.shape
    flat = out.reshape(B * H, N, d)
    res = np.zeros((len(items), block_l, d), np.float64)
    for i, (bh, qb) in enumerate(items):
        r0 = qb * block_l
        r1 = min(N, r0 + block_l)
        res[i, : r1 - r0] = flat[bh, r0:r1].double().cpu().numpy()
    return res


def heads_subset(t: torch.Tensor, bhs):
    """Slice [B,H,...] tensors down to the given flat (b*H + h) heads, keeping a 4-D shape."""
    B, H = t.shape[:2]
    return torch.stack([t[bh // H, bh % H] for bh in bhs]).unsqueeze(0)


def errors(got: np.ndarray, want: np.ndarray, mask=None):
    diff = np.abs(got - want)
    if mask is not None:
        diff = diff[mask]
    return float(diff.max()), float(diff.mean())


def oracle_items(q, k, v, items, *, block_l, G, seed=0, causal=False, scale=None):
    """Oracle output for work items (bh, qb), slicing one head at a time (bounded host memory).

    q: [B,H,N,d], k/v: [B,H_kv,N,d] torch tensors (any device/dtype: exact upcast to fp32)."""
    B, H, N, d = q.shape
    Hkv = k.shape[1]
    res = np.zeros((len(items), block_l, d), np.float64)
    by_head = {}
    for i, (bh, qb) in enumerate(items):
        by_head.setdefault(bh, []).append((i, qb))
    for bh, lst in by_head.items():
        b, h = divmod(bh, H)
        hk = h // (H // Hkv)
        qs = to_np32(q[b, h])[None, None]
        ks = to_np32(k[b, hk])[None, None]
        vs = to_np32(v[b, hk])[None, None]
        out = oracle.attn_items(qs, ks, vs, [(0, qb) for _, qb in lst], block_l=block_l, G=G,
                                seed=seed, causal=causal, scale=scale)
        for j, (i, _) in enumerate(lst):
            res[i] = out[j]
    return res


def valid_rows_mask(items, N, block_l, d):
    m = np.zeros((len(items), block_l, d), bool)
    for i, (_, qb) in enumerate(items):
        m[i, : min(block_l, N - qb * block_l)] = True
    return m
