"""DistrAttention (arXiv 2507.17245) forward hot path, B200-native (sm_100a).

Thin Python binding over the C-ABI in include/distr_attn.h: the functions below have the same
names as the C entry points and only marshal torch tensors (device memory + current stream) into
the da_params struct. Every compute step runs in libdistr_attn.so's CUDA kernels; there is no CPU
or PyTorch fallback (a missing library raises).
"""
from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _native
from ._native import DA_BF16, DA_F32, DaParams, DistrAttnError, check, last_launch_count

__all__ = [
    "distr_attn_fwd", "distr_attn_fwd_ex", "exact_attn_fwd_ex", "distr_attn_fwd_host",
    "distr_attn_hash", "distr_attn_projection", "distr_attn_workspace_size", "make_params",
    "DistrAttnError", "last_launch_count", "distr_attn_plan", "distr_attn_global_fwd_ex",
    "distr_attn_bwd_ex", "distr_attn_bwd_workspace_size", "distr_attn_choose",
]

_DT = {torch.bfloat16: DA_BF16, torch.float32: DA_F32}


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def make_params(q: torch.Tensor, k: torch.Tensor, *, block_l: int, group_size: int, seed: int = 0,
                causal: bool = False, scale: float = 0.0, lse=None, bucket_ids=None, perm=None,
                workspace=None, v=None, out=None, q_shard=None) -> DaParams:
    if q.dim() != 4 or k.dim() != 4:
        raise ValueError("q must be [B,H,N,d] and k/v [B,H_kv,N,d]")
    if k.shape[0] != q.shape[0] or k.shape[2:] != q.shape[2:] or k.dtype != q.dtype:
        raise ValueError(f"k {tuple(k.shape)} does not match q {tuple(q.shape)}")
    for t in (v, out):
        if t is not None and (t.dtype != q.dtype or
                              tuple(t.shape) != (tuple(k.shape) if t is v else tuple(q.shape))):
            raise ValueError("v must match k and out must match q (shape and dtype)")
    if q.dtype not in _DT:
        raise ValueError(f"unsupported dtype {q.dtype}")
    B, H, N, d = q.shape
    nqb = -(-N // block_l) if block_l > 0 else 0
    if lse is not None and (lse.dtype != torch.float32 or tuple(lse.shape) != (B, H, N)):
        raise ValueError(f"lse must be fp32 [B, H, N] = {(B, H, N)}")
    for name, t, dts in (("bucket_ids", bucket_ids, (torch.int16, torch.uint16)),
                         ("perm", perm, (torch.uint8,))):
        if t is not None and (t.dtype not in dts or t.numel() != B * H * nqb * d):
            raise ValueError(f"{name} must be {dts[0]} with B*H*ceil(N/block_l)*d = "
                             f"{B * H * nqb * d} elements")
    # every tensor the kernels touch: contiguous, and on the same side as q (device: q's device,
    # which must be the current one)
    for t in (q, k, v, out, lse, bucket_ids, perm, workspace):
        if t is None:
            continue
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")
        if t.is_cuda != q.is_cuda or (q.is_cuda and t.device != q.device):
            raise ValueError("all tensors must live on q's device (or all on the host)")
    if q.is_cuda and q.device.index != torch.cuda.current_device():
        raise ValueError(f"q is on {q.device} but the current device is cuda:{torch.cuda.current_device()}")
    p = DaParams()
    p.B, p.H, p.H_kv, p.N, p.d = B, H, k.shape[1], N, d
    p.block_l, p.group_size, p.seed = block_l, group_size, seed
    p.causal, p.scale, p.dtype = int(bool(causal)), float(scale), _DT[q.dtype]
    if workspace is not None:
        p.workspace, p.workspace_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    p.lse = None if lse is None else lse.data_ptr()
    p.bucket_ids = None if bucket_ids is None else bucket_ids.data_ptr()
    p.perm = None if perm is None else perm.data_ptr()
    if q_shard is not None:  # (offset, stride): Q-tile-pair sharding (shard.q_pair_shard)
        p.q_shard_offset, p.q_shard_stride = int(q_shard[0]), int(q_shard[1])
    return p


def _check_tensors(*ts):
    for t in ts:
        if t is not None and not t.is_contiguous():
            raise ValueError("tensors must be contiguous")


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def distr_attn_fwd_ex(q, k, v, out=None, *, block_l=128, group_size=2, seed=0, causal=False,
                      scale=0.0, lse=None, bucket_ids=None, perm=None, workspace=None, stream=None,
                      q_shard=None):
    """DistrAttention forward (device tensors, current torch stream). Returns `out`."""
    _check_tensors(q, k, v, out, lse)
    if out is None:
        out = torch.empty_like(q)
    p = make_params(q, k, block_l=block_l, group_size=group_size, seed=seed, causal=causal,
                    scale=scale, lse=lse, bucket_ids=bucket_ids, perm=perm, workspace=workspace,
                    v=v, out=out, q_shard=q_shard)
    check(_native.lib().distr_attn_fwd_ex(_ptr(q), _ptr(k), _ptr(v), _ptr(out), ctypes.byref(p),
                                          _stream(stream)))
    return out


def distr_attn_global_fwd_ex(q, k, v, out=None, *, group_size=2, seed=0, causal=False, scale=0.0,
                             lse=None, bucket_ids=None, perm=None, workspace=None, stream=None,
                             q_shard=None):
    """DistrAttention with one grouping per head (global LSH over all N rows). bf16 only;
    bucket_ids / perm exports are [B, H, 1, d]. Returns `out`."""
    _check_tensors(q, k, v, out, lse)
    B, H, N, d = q.shape
    if out is None:
        out = torch.empty_like(q)
    p = make_params(q, k, block_l=N, group_size=group_size, seed=seed, causal=causal,
                    scale=scale, lse=lse, bucket_ids=bucket_ids, perm=perm, workspace=workspace,
                    v=v, out=out, q_shard=q_shard)
    p.block_l = 128  # not used by the global variant (its tiles are 128 rows)
    check(_native.lib().distr_attn_global_fwd_ex(_ptr(q), _ptr(k), _ptr(v), _ptr(out), ctypes.byref(p),
                                                 _stream(stream)))
    return out


def distr_attn_bwd_ex(q, k, v, out, dout, lse, *, block_l=128, group_size=2, seed=0, causal=False,
                      scale=0.0, workspace=None, stream=None):
    """Backward of DistrAttention (grouping held constant, reading R18): returns (dq, dk, dv).
    `out` and `lse` ([B, H, N] fp32, natural log) come from the forward call with the same
    params; group_size=1 gives exact-attention gradients."""
    _check_tensors(q, k, v, out, dout, lse)
    if lse is None or lse.dtype != torch.float32 or tuple(lse.shape) != tuple(q.shape[:3]):
        raise ValueError("lse must be fp32 [B, H, N]")
    if dout.shape != q.shape or dout.dtype != q.dtype:
        raise ValueError("dout must match q")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    p = make_params(q, k, block_l=block_l, group_size=group_size, seed=seed, causal=causal,
                    scale=scale, v=v, out=out, workspace=workspace)
    check(_native.lib().distr_attn_bwd_ex(_ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(dout), _ptr(lse),
                                          _ptr(dq), _ptr(dk), _ptr(dv), ctypes.byref(p),
                                          _stream(stream)))
    return dq, dk, dv


def exact_attn_fwd_ex(q, k, v, out=None, *, block_l=128, causal=False, scale=0.0, lse=None,
                      workspace=None, stream=None, q_shard=None):
    """Exact attention on the same sm_100a tiling (reference point). Returns `out`."""
    _check_tensors(q, k, v, out, lse)
    if out is None:
        out = torch.empty_like(q)
    p = make_params(q, k, block_l=block_l, group_size=1, causal=causal, scale=scale, lse=lse,
                    workspace=workspace, v=v, out=out, q_shard=q_shard)
    check(_native.lib().exact_attn_fwd_ex(_ptr(q), _ptr(k), _ptr(v), _ptr(out), ctypes.byref(p),
                                          _stream(stream)))
    return out


def distr_attn_fwd(q, k, v, out, B, H, N, d, block_l, group_size, seed):
    """North-star signature (legacy default stream, bf16, H_kv = H, non-causal)."""
    for t in (q, k, v, out):
        if tuple(t.shape) != (B, H, N, d) or t.dtype != torch.bfloat16 or not t.is_contiguous():
            raise ValueError("distr_attn_fwd expects contiguous bf16 [B,H,N,d] q/k/v/out")
    check(_native.lib().distr_attn_fwd(_ptr(q), _ptr(k), _ptr(v), _ptr(out), B, H, N, d, block_l,
                                       group_size, seed))
    return out


def distr_attn_fwd_host(q, k, v, out=None, *, block_l=128, group_size=2, seed=0, causal=False,
                        scale=0.0, lse=None, bucket_ids=None, perm=None, stream=None, q_shard=None):
    """Forward over HOST (ideally pinned) tensors: H2D + kernels + D2H inside the C call."""
    for t in (q, k, v):
        if t.is_cuda:
            raise ValueError("distr_attn_fwd_host takes host tensors")
    _check_tensors(q, k, v, out, lse)
    if out is None:
        out = torch.empty_like(q)
    p = make_params(q, k, block_l=block_l, group_size=group_size, seed=seed, causal=causal,
                    scale=scale, lse=lse, bucket_ids=bucket_ids, perm=perm, v=v, out=out,
                    q_shard=q_shard)
    check(_native.lib().distr_attn_fwd_host(_ptr(q), _ptr(k), _ptr(v), _ptr(out), ctypes.byref(p),
                                            _stream(stream)))
    return out


def distr_attn_hash(q, *, block_l=128, group_size=2, seed=0, stream=None):
    """LSH step only: returns (bucket_ids uint16-as-int16 [B,H,nqb,d], perm uint8 [B,H,nqb,d])."""
    _check_tensors(q)
    B, H, N, d = q.shape
    nqb = -(-N // block_l)
    buckets = torch.empty((B, H, nqb, d), dtype=torch.int16, device=q.device)
    perm = torch.empty((B, H, nqb, d), dtype=torch.uint8, device=q.device)
    p = make_params(q, q, block_l=block_l, group_size=group_size, seed=seed, bucket_ids=buckets,
                    perm=perm)
    check(_native.lib().distr_attn_hash(_ptr(q), ctypes.byref(p), _stream(stream)))
    return buckets, perm


def distr_attn_projection(seed: int, block_l: int) -> np.ndarray:
    out = np.empty((16, block_l), dtype=np.float32)
    check(_native.lib().distr_attn_projection(seed, block_l, out.ctypes.data_as(ctypes.c_void_p)))
    return out


def distr_attn_workspace_size(q_shape, kv_heads, *, block_l=128, group_size=2,
                              dtype=torch.bfloat16) -> int:
    B, H, N, d = q_shape
    p = DaParams()
    p.B, p.H, p.H_kv, p.N, p.d = B, H, kv_heads, N, d
    p.block_l, p.group_size, p.dtype = block_l, group_size, _DT[dtype]
    return int(_native.lib().distr_attn_workspace_size(ctypes.byref(p)))


def distr_attn_bwd_workspace_size(q_shape, kv_heads, *, block_l=128, group_size=2,
                                  dtype=torch.bfloat16) -> int:
    B, H, N, d = q_shape
    p = DaParams()
    p.B, p.H, p.H_kv, p.N, p.d = B, H, kv_heads, N, d
    p.block_l, p.group_size, p.dtype = block_l, group_size, _DT[dtype]
    return int(_native.lib().distr_attn_bwd_workspace_size(ctypes.byref(p)))


def distr_attn_plan(N: int, d: int, *, block_l: int = 128, group_size: int = 2, distr: bool = True) -> dict:
    """Block-size planner (include/distr_attn.h distr_attn_plan; §3.3.1 P:320-369 re-derived for
    tcgen05/TMEM). Host-only: no GPU needed."""
    out = _native.DaPlan()
    check(_native.lib().distr_attn_plan(N, d, block_l, group_size, int(distr), ctypes.byref(out)))
    return {name: getattr(out, name) for name, _ in _native.DaPlan._fields_}


def distr_attn_choose(B: int, H: int, H_kv: int, N: int, d: int, *, causal: bool = False,
                      max_group_size: int = 4, clk_mhz: float = 0.0) -> dict:
    """Planner choice (include/distr_attn.h distr_attn_choose): exact kernel or DistrAttention
    with (block_l, G* <= max_group_size), by predicted forward time on one B200. Host-only."""
    out = _native.DaChoice()
    check(_native.lib().distr_attn_choose(B, H, H_kv, N, d, int(bool(causal)), max_group_size,
                                          float(clk_mhz), ctypes.byref(out)))
    return {name: getattr(out, name) for name, _ in _native.DaChoice._fields_}


def default_scale(d: int) -> float:
    return 1.0 / math.sqrt(d)
