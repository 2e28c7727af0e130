"""Pins for the backward oracle (oracle/backward.py, reading R18), CPU only."""
import numpy as np
import pytest
import torch

import oracle
from oracle.backward import attn_bwd, groups_of


def draw(B, H, Hkv, N, d, seed, grid=None):
    g = np.random.default_rng(seed)
    if grid:  # values on a 2^-grid lattice: q ± 2^-grid stays exact in fp32 (finite differences)
        f = lambda *s: np.round(g.standard_normal(s) * 2 ** grid) / 2 ** grid
    else:
        f = lambda *s: g.standard_normal(s)
    return (f(B, H, N, d).astype(np.float32), f(B, Hkv, N, d).astype(np.float32),
            f(B, Hkv, N, d).astype(np.float32), g.standard_normal((B, H, N, d)))


def torch_reference(q, k, v, do, causal, scale):
    """Exact attention gradients by torch.autograd in float64 (independent of the oracle)."""
    q, k, v = (torch.tensor(x, dtype=torch.float64, requires_grad=True) for x in (q, k, v))
    rep = q.shape[1] // k.shape[1]
    ke, ve = k.repeat_interleave(rep, dim=1), v.repeat_interleave(rep, dim=1)
    s = scale * q @ ke.transpose(-1, -2)
    if causal:
        n = q.shape[2]
        s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool), 1), float("-inf"))
    o = torch.softmax(s, dim=-1) @ ve
    (o * torch.tensor(do)).sum().backward()
    return q.grad.numpy(), k.grad.numpy(), v.grad.numpy(), o.detach().numpy()


@pytest.mark.parametrize("causal", [False, True])
def test_exact_gradients_match_torch_autograd(causal):
    q, k, v, do = draw(1, 4, 2, 70, 16, 1)
    dq, dk, dv, o = attn_bwd(q, k, v, do, block_l=32, G=0, causal=causal)
    rq, rk, rv, ro = torch_reference(q, k, v, do, causal, 1 / 4)
    for a, b in ((o, ro), (dq, rq), (dk, rk), (dv, rv)):
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-12)


def test_group_size_one_equals_exact():
    q, k, v, do = draw(1, 2, 2, 50, 16, 2)
    a = attn_bwd(q, k, v, do, block_l=16, G=1, causal=True)
    b = attn_bwd(q, k, v, do, block_l=16, G=0, causal=True)
    for x, y in zip(a, b):
        np.testing.assert_allclose(x, y, rtol=1e-11, atol=1e-13)


def test_forward_matches_c_oracle():
    q, k, v, do = draw(1, 2, 1, 45, 16, 3)
    o = attn_bwd(q, k, v, do, block_l=16, G=2, seed=5, causal=True)[3]
    ref = oracle.attn_full(q, k, v, block_l=16, G=2, seed=5, causal=True)
    np.testing.assert_allclose(o, ref, rtol=1e-10, atol=1e-12)


def fixed_group_forward(q, k, v, perms, block_l, G, scale, causal):
    """Forward of DistrAttention with the given per-block permutations held fixed: Ŝ from the C
    oracle's Eq. 2 routine (oracle_grouped_scores), softmax and PV in float64."""
    B, H, N, d = q.shape
    o = np.zeros(q.shape)
    for b in range(B):
        for h in range(H):
            hk = h // (H // k.shape[1])
            for qb in range(-(-N // block_l)):
                r0, r1 = qb * block_l, min(N, (qb + 1) * block_l)
                s = oracle.grouped_scores(q[b, h, r0:r1], k[b, hk], perms[b, h, qb], G, scale)
                if causal:
                    s = np.where(np.arange(N)[None, :] > np.arange(r0, r1)[:, None], -np.inf, s)
                p = np.exp(s - s.max(axis=1, keepdims=True))
                o[b, h, r0:r1] = (p / p.sum(axis=1, keepdims=True)) @ v[b, hk].astype(np.float64)
    return o


def test_finite_differences_with_fixed_grouping():
    # f = sum(O * W): central differences of the C-oracle forward (grouping held fixed, R18)
    q, k, v, W = draw(1, 2, 1, 40, 16, 4, grid=6)
    block_l, G, scale, causal = 16, 2, 0.25, True
    perms = oracle.hash_all(q, block_l, 0)[1]
    dq, dk, dv, _ = attn_bwd(q, k, v, W, block_l=block_l, G=G, causal=causal, scale=scale)
    f = lambda q_, k_, v_: float((fixed_group_forward(q_, k_, v_, perms, block_l, G, scale, causal) * W).sum())
    rng = np.random.default_rng(0)
    eps = 2.0 ** -6
    for name, x, grad in (("q", q, dq), ("k", k, dk), ("v", v, dv)):
        for _ in range(12):
            idx = tuple(rng.integers(0, s) for s in x.shape)
            xp, xm = x.copy(), x.copy()
            xp[idx] += eps
            xm[idx] -= eps
            args_p = [xp if n == name else y for n, y in (("q", q), ("k", k), ("v", v))]
            args_m = [xm if n == name else y for n, y in (("q", q), ("k", k), ("v", v))]
            fd = (f(*args_p) - f(*args_m)) / (2 * eps)
            assert abs(fd - grad[idx]) <= 2e-3 * max(1.0, abs(grad[idx])), (name, idx, fd, grad[idx])


@pytest.mark.parametrize("G", [2, 4])
def test_duplicated_columns_fold_exact_gradients(G):
    # duplicated Q columns: forward == exact (Eq. 1); dK, dV equal the exact ones and dQ holds, on
    # each representative column, the sum of the exact gradient over its group (zero elsewhere)
    g = np.random.default_rng(5)
    base = g.standard_normal((1, 2, 48, 32 // G)).astype(np.float32)
    q = np.repeat(base, G, axis=-1)
    k = g.standard_normal((1, 2, 48, 32)).astype(np.float32)
    v = g.standard_normal((1, 2, 48, 32)).astype(np.float32)
    do = g.standard_normal((1, 2, 48, 32))
    dq, dk, dv, o = attn_bwd(q, k, v, do, block_l=16, G=G)
    eq, ek, ev, eo = attn_bwd(q, k, v, do, block_l=16, G=0)
    np.testing.assert_allclose(o, eo, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dk, ek, rtol=1e-9, atol=1e-11)
    np.testing.assert_allclose(dv, ev, rtol=1e-10, atol=1e-12)
    perms = oracle.hash_all(q, 16, 0)[1]
    for qb in range(3):
        for h in range(2):
            for rep, mem in groups_of(perms[0, h, qb], G):
                rows = slice(qb * 16, qb * 16 + 16)
                np.testing.assert_allclose(dq[0, h, rows, rep], eq[0, h, rows][:, mem].sum(axis=1),
                                           rtol=1e-9, atol=1e-11)
                for c in mem:
                    if c != rep:
                        assert np.all(dq[0, h, rows, c] == 0)
