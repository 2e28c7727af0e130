"""ctypes binding of libdistr_attn.so (include/distr_attn.h). Argument marshalling only.

The library is the product: there is no fallback. If libdistr_attn.so is missing or fails to load
this module raises; every compute step runs in the library's CUDA kernels.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdistr_attn.so")

DA_OK, DA_ERR_INVALID, DA_ERR_PRECONDITION, DA_ERR_CUDA = 0, 1, 2, 3
DA_BF16, DA_F32 = 0, 1

# Every symbol include/distr_attn.h declares.
EXPORTED = (
    "distr_attn_init_params", "distr_attn_fwd", "distr_attn_fwd_ex", "distr_attn_fwd_host",
    "exact_attn_fwd_ex", "distr_attn_hash", "distr_attn_projection", "distr_attn_workspace_size",
    "distr_attn_status_string", "distr_attn_last_error", "distr_attn_last_launch_count",
    "distr_attn_set_profile_events", "distr_attn_set_trace", "distr_attn_plan",
    "distr_attn_global_fwd_ex", "distr_attn_bwd_ex", "distr_attn_bwd_workspace_size",
    "distr_attn_choose",
)


class DaParams(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int), ("H", ctypes.c_int), ("H_kv", ctypes.c_int), ("N", ctypes.c_int),
        ("d", ctypes.c_int), ("block_l", ctypes.c_int), ("group_size", ctypes.c_int),
        ("seed", ctypes.c_ulonglong), ("causal", ctypes.c_int), ("scale", ctypes.c_float),
        ("dtype", ctypes.c_int), ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_size_t), ("lse", ctypes.c_void_p),
        ("bucket_ids", ctypes.c_void_p), ("perm", ctypes.c_void_p),
        ("q_shard_offset", ctypes.c_int), ("q_shard_stride", ctypes.c_int),
    ]


class DaPlan(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "tile_m", "tiles_per_cta", "tile_n", "s_width", "kv_stages", "khat_stages", "threads",
        "smem_bytes", "tmem_cols", "m_max_tmem", "ctas")] + [(n, ctypes.c_double) for n in (
        "mma_clk_per_tile", "exp_clk_per_tile", "fusion_smem_bytes_per_tile", "hbm_bytes_paper",
        "hbm_bytes_b200")]


class DaChoice(ctypes.Structure):
    _fields_ = [("distr", ctypes.c_int), ("block_l", ctypes.c_int), ("group_size", ctypes.c_int),
                ("predicted_us", ctypes.c_double), ("predicted_exact_us", ctypes.c_double),
                ("predicted_distr_us", ctypes.c_double)]


class DistrAttnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load libdistr_attn.so (built in-tree by paper_2507_17245_b200.build). Raises if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} not found: build it with `python -m paper_2507_17245_b200.build` "
                    "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            vp, i32, P = ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(DaParams)
            L.distr_attn_init_params.argtypes = [P, i32, i32, i32, i32, i32, i32, ctypes.c_ulonglong]
            L.distr_attn_fwd.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32,
                                         ctypes.c_ulonglong]
            for name in ("distr_attn_fwd_ex", "exact_attn_fwd_ex", "distr_attn_fwd_host",
                         "distr_attn_global_fwd_ex"):
                getattr(L, name).argtypes = [vp, vp, vp, vp, P, vp]
            L.distr_attn_hash.argtypes = [vp, P, vp]
            L.distr_attn_projection.argtypes = [ctypes.c_ulonglong, i32, vp]
            L.distr_attn_workspace_size.argtypes = [P]
            L.distr_attn_workspace_size.restype = ctypes.c_size_t
            L.distr_attn_bwd_workspace_size.argtypes = [P]
            L.distr_attn_bwd_workspace_size.restype = ctypes.c_size_t
            L.distr_attn_status_string.argtypes = [i32]
            L.distr_attn_status_string.restype = ctypes.c_char_p
            L.distr_attn_last_error.restype = ctypes.c_char_p
            L.distr_attn_last_launch_count.restype = i32
            L.distr_attn_set_profile_events.argtypes = [vp, vp, vp]
            L.distr_attn_set_trace.argtypes = [vp]
            L.distr_attn_bwd_ex.argtypes = [vp] * 9 + [P, vp]
            L.distr_attn_plan.argtypes = [i32, i32, i32, i32, i32, ctypes.POINTER(DaPlan)]
            L.distr_attn_choose.argtypes = [i32, i32, i32, i32, i32, i32, i32, ctypes.c_double,
                                            ctypes.POINTER(DaChoice)]
            _lib = L
    return _lib


def check(status: int) -> None:
    if status != DA_OK:
        L = lib()
        detail = L.distr_attn_last_error().decode()
        raise DistrAttnError(status, f"{L.distr_attn_status_string(status).decode()}: {detail}")


def last_launch_count() -> int:
    return int(lib().distr_attn_last_launch_count())
