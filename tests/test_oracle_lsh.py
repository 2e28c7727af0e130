"""Pins for the oracle's LSH steps. CPU only.

Each test checks the oracle against something other than itself: closed forms of the Gray code,
exact algebraic invariances of an fp32 fma chain, an independent fp64 numpy projection, the
paper's Fig. 5 worked example, and distribution statistics for the projection matrix.
"""
import numpy as np
import pytest
from scipy import stats

import oracle


def gray_encode(b):
    """Textbook reflected-binary Gray codeword of rank b (closed form)."""
    return b ^ (b >> 1)


# ---------------------------------------------------------------- Gray rank (reading R2)
def test_gray_rank_spec_examples():
    # 0b0000 -> 0, 0b0001 -> 1, 0b0010 -> 3 ; and 0b0011 -> 2 (reflected sequence)
    assert [oracle.gray_rank(p) for p in (0, 1, 2, 3)] == [0, 1, 3, 2]


def test_gray_rank_is_inverse_of_reflected_code_and_adjacent():
    ranks = np.array([oracle.gray_rank(p) for p in range(1 << 16)])
    assert sorted(ranks.tolist()) == list(range(1 << 16))  # bijection on 2^16
    for r in range(1 << 16):
        assert ranks[gray_encode(r)] == r
    # consecutive ranks <-> patterns at Hamming distance 1 (the property P:292 relies on)
    inv = np.empty(1 << 16, dtype=np.int64)
    inv[ranks] = np.arange(1 << 16)
    x = inv[1:] ^ inv[:-1]
    assert np.all((x & (x - 1)) == 0) and np.all(x != 0)


# ---------------------------------------------------------------- projection (R4)
def test_projection_is_standard_normal_and_deterministic():
    p = oracle.projection(0, 128)
    assert p.shape == (16, 128) and p.dtype == np.float32
    assert np.array_equal(p, oracle.projection(0, 128))
    assert not np.array_equal(p, oracle.projection(1, 128))
    big = np.concatenate([oracle.projection(s, 128).ravel() for s in range(32)]).astype(np.float64)
    n = big.size
    assert abs(big.mean()) < 4.0 / np.sqrt(n)
    assert abs(big.var() - 1.0) < 6.0 * np.sqrt(2.0 / n)
    assert stats.kstest(big, "norm").pvalue > 1e-3
    # consecutive Box-Muller pairs must be uncorrelated
    assert abs(np.corrcoef(big[0::2], big[1::2])[0, 1]) < 4.0 / np.sqrt(n / 2)


# ---------------------------------------------------------------- hashing (R3/R5/R6/R9)
def test_zero_column_hashes_to_zero():
    # no positive projection -> pattern 0 -> bucket 0; +0 and -0 both give bit 0 (R5)
    proj = oracle.projection(3, 64)
    q = np.zeros((64, 8), np.float32)
    q[:, 1] = -0.0
    assert np.all(oracle.hash_block(q, proj) == 0)


def test_hash_invariant_under_power_of_two_scaling():
    rng = np.random.default_rng(0)
    proj = oracle.projection(5, 128)
    q = rng.standard_normal((128, 128)).astype(np.float32)
    h = oracle.hash_block(q, proj)
    for s in (2.0 ** -20, 0.5, 4.0, 2.0 ** 30):
        assert np.array_equal(oracle.hash_block(q * np.float32(s), proj), h)


def test_hash_sign_flip_complements_pattern():
    rng = np.random.default_rng(1)
    proj = oracle.projection(11, 64)
    q = rng.standard_normal((64, 64)).astype(np.float32)
    a = np.array([gray_encode(int(b)) for b in oracle.hash_block(q, proj)])
    b = np.array([gray_encode(int(b)) for b in oracle.hash_block(-q, proj)])
    assert np.all(a ^ b == 0xFFFF)


def test_hash_matches_fp64_projection_on_margin_columns():
    """Independent check of indexing P[k][r], bit order (bit k = row k, LSB first) and y > 0."""
    rng = np.random.default_rng(2)
    for l, rows in ((64, 64), (128, 128), (64, 5), (128, 77)):
        proj = oracle.projection(7, l)
        q = rng.standard_normal((rows, 128)).astype(np.float32)
        y = proj[:, :rows].astype(np.float64) @ q.astype(np.float64)  # [16, d], BLAS order
        margin = np.abs(y).min(axis=0) > 1e-3
        want = ((y > 0).astype(np.int64) << np.arange(16)[:, None]).sum(axis=0)
        got = np.array([gray_encode(int(b)) for b in oracle.hash_block(q, proj)])
        assert margin.sum() > 50
        assert np.array_equal(got[margin], want[margin])


def test_ragged_block_equals_zero_padded_block():
    rng = np.random.default_rng(3)
    proj = oracle.projection(9, 64)
    q5 = rng.standard_normal((5, 64)).astype(np.float32)
    pad = np.zeros((64, 64), np.float32)
    pad[:5] = q5
    assert np.array_equal(oracle.hash_block(q5, proj), oracle.hash_block(pad, proj))


def test_hash_all_matches_per_block():
    rng = np.random.default_rng(4)
    q = rng.uniform(size=(2, 3, 197, 64)).astype(np.float32)  # U(0,1): many tied buckets
    buckets, perm = oracle.hash_all(q, 64, 0)
    proj = oracle.projection(0, 64)
    assert buckets.shape == (2, 3, 4, 64)
    for b in range(2):
        for h in range(3):
            for qb in range(4):
                blk = q[b, h, qb * 64:(qb + 1) * 64]
                hb = oracle.hash_block(blk, proj)
                assert np.array_equal(buckets[b, h, qb], hb)
                assert np.array_equal(perm[b, h, qb], np.argsort(hb, kind="stable"))


# ---------------------------------------------------------------- sort (Fig. 5)
def test_fig5_permutation():
    # Fig. 5: hashes sorted to {h3, h2, h1, h4} -> permutation {3, 2, 1, 4} (1-based)
    h = np.array([30, 20, 10, 40], np.uint16)
    assert (oracle.sort_perm(h) + 1).tolist() == [3, 2, 1, 4]


def test_sort_is_stable_and_identity_on_ties():
    assert oracle.sort_perm(np.full(64, 7, np.uint16)).tolist() == list(range(64))
    rng = np.random.default_rng(5)
    for _ in range(50):
        h = rng.integers(0, 6, size=128).astype(np.uint16)
        assert np.array_equal(oracle.sort_perm(h), np.argsort(h, kind="stable"))
