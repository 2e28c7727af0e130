"""CPU ORACLE for the DistrAttention backward pass — TEST INFRASTRUCTURE ONLY (same rules as
oracle.c: only tests/, smoke() and bench.py's baseline legs may import it; it shares no code with
paper_2507_17245_b200/).

Reading R18. The paper fine-tunes with DistrAttention but
never defines gradients through LSH, sampling and fusion. The grouping is a piecewise-constant
function of Q (a hash), so its derivative is zero almost everywhere: the permutation of every Q
block is treated as a constant. Eq. 2 then reads Ŝ = scale · Q̂ K̂ᵀ with
Q̂ = Q[:, rep] (rep_j = first member of group j, R10) and K̂ = K M (M the d × d/G* 0/1 grouping
matrix), followed by the standard softmax attention (§2.1). Its backward:

    dV  = Pᵀ dO
    dP  = dO Vᵀ ;  dŜ = P ∘ (dP − rowsum(dO ∘ O))
    dQ̂  = scale · dŜ K̂   →  dQ[:, rep_j] = dQ̂[:, j], zero in non-representative columns
    dK̂  = scale · dŜᵀ Q̂  →  dK[:, c] = dK̂[:, j(c)] for every member c of group j

summed over the Q blocks (each with its own grouping, §3.3) and over the query heads
that share a KV head (GQA, R11). Causal: masked after the approximation (R11). Everything is
float64 numpy, one (b, h, Q block) at a time, in the order written above.
G = 0 selects exact attention (identity grouping, no sampling).

Pins (tests/test_oracle_backward.py): G = 0 against torch.autograd of an fp64 softmax-attention
written independently; finite differences of the C oracle's forward with the grouping held
fixed (oracle.grouped_scores); the duplicated-column identity (dQ folds the exact gradient onto
representatives, dK and dV equal the exact ones).
"""
from __future__ import annotations

import numpy as np

from . import _f32, hash_all


def groups_of(perm: np.ndarray, G: int):
    """[(rep, members)] per group j from a block's permutation (R10)."""
    d = perm.shape[0]
    return [(int(perm[j * G]), [int(c) for c in perm[j * G:(j + 1) * G]]) for j in range(d // G)]


def attn_bwd(q, k, v, do, *, block_l: int, G: int, seed: int = 0, causal: bool = False,
             scale: float | None = None):
    """Gradients (dq, dk, dv) and the forward output o, float64, for DistrAttention (G >= 1) or
    exact attention (G = 0). q, do: [B,H,N,d]; k, v: [B,H_kv,N,d]."""
    q, k, v = _f32(q).astype(np.float64), _f32(k).astype(np.float64), _f32(v).astype(np.float64)
    do = np.asarray(do, dtype=np.float64)
    B, H, N, d = q.shape
    H_kv = k.shape[1]
    if scale is None:
        scale = 1.0 / float(np.sqrt(d))  # R12
    nqb = -(-N // block_l)
    perms = hash_all(_f32(q), block_l, seed)[1] if G >= 1 else None
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    o = np.zeros_like(q)
    keys = np.arange(N)
    for b in range(B):
        for h in range(H):
            hk = h // (H // H_kv)
            K, V = k[b, hk], v[b, hk]
            for qb in range(nqb):
                r0, r1 = qb * block_l, min(N, (qb + 1) * block_l)
                Q, dO = q[b, h, r0:r1], do[b, h, r0:r1]
                if G >= 1:
                    grp = groups_of(perms[b, h, qb], G)
                    Qh = np.stack([Q[:, rep] for rep, _ in grp], axis=1)                # Q̂
                    Kh = np.stack([K[:, mem].sum(axis=1) for _, mem in grp], axis=1)  # K̂
                else:
                    grp, Qh, Kh = None, Q, K
                S = scale * (Qh @ Kh.T)
                if causal:
                    S = np.where(keys[None, :] > np.arange(r0, r1)[:, None], -np.inf, S)
                S = S - S.max(axis=1, keepdims=True)
                P = np.exp(S)
                P /= P.sum(axis=1, keepdims=True)
                O = P @ V
                o[b, h, r0:r1] = O
                dv[b, hk] += P.T @ dO
                dP = dO @ V.T
                dS = P * (dP - (dO * O).sum(axis=1, keepdims=True))
                dQh = scale * (dS @ Kh)
                dKh = scale * (dS.T @ Qh)
                if G >= 1:
                    for j, (rep, mem) in enumerate(grp):
                        dq[b, h, r0:r1, rep] += dQh[:, j]
                        for c in mem:
                            dk[b, hk, :, c] += dKh[:, j]
                else:
                    dq[b, h, r0:r1] += dQh
                    dk[b, hk] += dKh
    return dq, dk, dv, o
