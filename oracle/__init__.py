"""CPU oracle for DistrAttention (arXiv 2507.17245) — TEST INFRASTRUCTURE, NOT THE PRODUCT.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. It wraps ``oracle/oracle.c`` (plain C,
OpenMP over work items, fp32 fma-chain hashing, fp64 everything else) through ctypes and shares
no code with ``paper_2507_17245_b200`` (the CUDA product path), which never imports it.

Every function cites the PAPER.md passage it follows (see oracle.c). Parity pins live in
``tests/test_oracle_*.py``; all oracle functions are pinned (none is "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

NPRIME = 16


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -fopenmp -ffp-contract=off, no fast-math)."""
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)):
        return _LIB_PATH
    cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
           "-fPIC", "-shared", "-o", _LIB_PATH + ".tmp", _SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            u64, i32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
            L.oracle_projection.argtypes = [u64, i32, vp]
            L.oracle_projection.restype = None
            L.oracle_gray_rank.argtypes = [ctypes.c_uint32]
            L.oracle_gray_rank.restype = ctypes.c_uint32
            L.oracle_hash_block.argtypes = [vp, i32, i32, i32, vp, i32, vp]
            L.oracle_hash_block.restype = None
            L.oracle_sort_perm.argtypes = [vp, i32, vp]
            L.oracle_sort_perm.restype = None
            L.oracle_hash.argtypes = [vp, i32, i32, i32, i32, i32, u64, vp, vp]
            L.oracle_hash.restype = i32
            L.oracle_grouped_scores.argtypes = [vp, i32, i32, vp, i32, i32, i32, i32, vp,
                                                ctypes.c_double, vp]
            L.oracle_grouped_scores.restype = None
            L.oracle_distr_scores.argtypes = [vp, i32, i32, vp, i32, i32, i32, i32, i32, u64,
                                              ctypes.c_double, vp, vp]
            L.oracle_distr_scores.restype = i32
            L.oracle_attn_items.argtypes = [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, u64,
                                            i32, ctypes.c_double, vp, i32, vp, vp]
            L.oracle_attn_items.restype = i32
            L.oracle_num_threads.restype = i32
            L.oracle_set_num_threads.argtypes = [i32]
            L.oracle_ftz_daz_clear.restype = i32
            _lib = L
    return _lib


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def projection(seed: int, block_l: int) -> np.ndarray:
    """[16, block_l] fp32 projection matrix (reading R4)."""
    out = np.empty((NPRIME, block_l), dtype=np.float32)
    lib().oracle_projection(seed, block_l, _ptr(out))
    return out


def gray_rank(pattern: int) -> int:
    """Rank of a bit pattern in the reflected Gray sequence (reading R2)."""
    return int(lib().oracle_gray_rank(pattern))


def hash_block(q_block, proj: np.ndarray) -> np.ndarray:
    """Bucket ids (uint16 [d]) of one Q block [rows, d] (reading R5/R6/R9)."""
    q_block = _f32(q_block)
    rows, d = q_block.shape
    proj = _f32(proj)
    block_l = proj.shape[1]
    assert rows <= block_l
    out = np.empty(d, dtype=np.uint16)
    lib().oracle_hash_block(_ptr(q_block), rows, d, d, _ptr(proj), block_l, _ptr(out))
    return out


def sort_perm(buckets) -> np.ndarray:
    """Stable ascending permutation of bucket ids (Fig. 5)."""
    b = np.ascontiguousarray(np.asarray(buckets, dtype=np.uint16))
    out = np.empty(b.shape[0], dtype=np.uint8)
    lib().oracle_sort_perm(_ptr(b), b.shape[0], _ptr(out))
    return out


def hash_all(q, block_l: int, seed: int):
    """Bucket ids and perms for every Q block of q [B, H, N, d] -> ([B,H,nqb,d] u16, u8)."""
    q = _f32(q)
    B, H, N, d = q.shape
    nqb = -(-N // block_l)
    buckets = np.empty((B, H, nqb, d), dtype=np.uint16)
    perm = np.empty((B, H, nqb, d), dtype=np.uint8)
    rc = lib().oracle_hash(_ptr(q), B, H, N, d, block_l, seed, _ptr(buckets), _ptr(perm))
    if rc:
        raise ValueError(f"oracle_hash failed ({rc})")
    return buckets, perm


def grouped_scores(q_block, k, perm, G: int, scale: float = 1.0) -> np.ndarray:
    """Ŝ = scale * Q̂ K̂^T for a given permutation (Eq. 2), double [rows, nk]."""
    q_block, k = _f32(q_block), _f32(k)
    rows, d = q_block.shape
    nk = k.shape[0]
    perm = np.ascontiguousarray(np.asarray(perm, dtype=np.uint8))
    out = np.empty((rows, nk), dtype=np.float64)
    lib().oracle_grouped_scores(_ptr(q_block), rows, d, _ptr(k), nk, d, d, G, _ptr(perm),
                                float(scale), _ptr(out))
    return out


def distr_scores(q_block, k, block_l: int, G: int, seed: int, scale: float = 1.0):
    """Hash + sort + Eq. 2 for one Q block: returns (Ŝ [rows, nk] double, perm [d])."""
    q_block, k = _f32(q_block), _f32(k)
    rows, d = q_block.shape
    nk = k.shape[0]
    out = np.empty((rows, nk), dtype=np.float64)
    perm = np.empty(d, dtype=np.uint8)
    rc = lib().oracle_distr_scores(_ptr(q_block), rows, d, _ptr(k), nk, d, d, block_l, G, seed,
                                   float(scale), _ptr(out), _ptr(perm))
    if rc:
        raise ValueError(f"oracle_distr_scores failed ({rc})")
    return out, perm


def attn_items(q, k, v, items, *, block_l: int, G: int, seed: int = 0, causal: bool = False,
               scale: float | None = None, want_lse: bool = False):
    """Attention output (double) for work items [(bh, qb), ...].

    G == 0 -> exact attention (§2.1); G >= 1 -> DistrAttention (Eq. 2 + §3.3).
    q: [B,H,N,d], k/v: [B,H_kv,N,d] (fp32 arrays; exact upcasts of the kernel inputs).
    Returns out [n_items, block_l, d] (rows past N are zero) and optionally lse [n_items, block_l].
    """
    q, k, v = _f32(q), _f32(k), _f32(v)
    B, H, N, d = q.shape
    H_kv = k.shape[1]
    if scale is None:
        scale = 1.0 / float(np.sqrt(d))  # reading R12: 1/sqrt(original d)
    it = np.ascontiguousarray(np.asarray(items, dtype=np.int32).reshape(-1, 2))
    n = it.shape[0]
    out = np.zeros((n, block_l, d), dtype=np.float64)
    lse = np.full((n, block_l), np.nan, dtype=np.float64) if want_lse else None
    rc = lib().oracle_attn_items(_ptr(q), _ptr(k), _ptr(v), B, H, H_kv, N, d, block_l, G, seed,
                                 int(bool(causal)), float(scale), _ptr(it), n, _ptr(out),
                                 _ptr(lse) if lse is not None else None)
    if rc:
        raise ValueError(f"oracle_attn_items failed ({rc})")
    return (out, lse) if want_lse else out


def attn_full(q, k, v, *, block_l: int, G: int, seed: int = 0, causal: bool = False,
              scale: float | None = None) -> np.ndarray:
    """Whole-tensor attention [B,H,N,d] double (all Q blocks of all heads)."""
    q = _f32(q)
    B, H, N, d = q.shape
    nqb = -(-N // block_l)
    items = [(bh, qb) for bh in range(B * H) for qb in range(nqb)]
    out = attn_items(q, k, v, items, block_l=block_l, G=G, seed=seed, causal=causal, scale=scale)
    out = out.reshape(B * H, nqb * block_l, d)[:, :N, :]
    return out.reshape(B, H, N, d)


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def ftz_daz_clear() -> bool:
    return bool(lib().oracle_ftz_daz_clear())
