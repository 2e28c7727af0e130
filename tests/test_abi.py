"""C-ABI checks that need no GPU: the library loads, exports every symbol include/distr_attn.h
declares, validates arguments before touching CUDA, and its host-side projection generator is
bit-identical to the oracle's independent implementation (reading R4)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import paper_2507_17245_b200 as da
from paper_2507_17245_b200 import _native
from paper_2507_17245_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build()
    return _native.lib()


def header_functions():
    src = "".join(open(os.path.join(ROOT, "include", h)).read()
                  for h in sorted(os.listdir(os.path.join(ROOT, "include"))) if h.endswith(".h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(\w+)\s*\(", src, flags=re.M))


def test_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) == 18, names
    assert names == set(_native.EXPORTED)
    for n in names:
        assert hasattr(L, n), n


def test_so_contains_sm100a_tcgen05_code(L):
    import subprocess
    sass = subprocess.run(["cuobjdump", "-sass", _native.LIB_PATH], capture_output=True,
                          text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM", "STTM", "FFMA2"):
        assert mnemonic in sass, mnemonic
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)  # no legacy mma.sync path


@pytest.mark.parametrize("seed,l", [(0, 64), (0, 128), (123456789, 128), (2**63 + 5, 64)])
def test_projection_bit_identical_to_oracle(L, seed, l):
    a = da.distr_attn_projection(seed, l)
    b = oracle.projection(seed, l)
    assert a.view(np.uint32).tobytes() == b.view(np.uint32).tobytes()


def params(**kw):
    p = _native.DaParams()
    L = _native.lib()
    L.distr_attn_init_params(ctypes.byref(p), kw.pop("B", 1), kw.pop("H", 2), kw.pop("N", 256),
                             kw.pop("d", 64), kw.pop("block_l", 64), kw.pop("G", 2), 0)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


FAKE = ctypes.c_void_p(0x1000)


@pytest.mark.parametrize("kw,status", [
    (dict(B=0), 1), (dict(N=-1), 1), (dict(H=3, H_kv=2), 1), (dict(dtype=7), 1),
    (dict(causal=2), 1), (dict(d=96), 2), (dict(d=64, G=3), 2), (dict(G=8), 2),
    (dict(block_l=32), 2), (dict(d=64, block_l=64, G=1), 0), (dict(d=128, block_l=64, G=1), 2),
    (dict(d=128, block_l=128, G=8), 0), (dict(d=128, block_l=64, G=8), 0), (dict(d=128, G=16), 2),
    (dict(d=32, block_l=128, G=2), 0), (dict(d=32, block_l=64, G=2), 0), (dict(d=32, G=4), 2),
    (dict(d=128, block_l=256, G=2), 0), (dict(d=64, block_l=256, G=4), 0), (dict(d=32, block_l=256, G=2), 0),
    (dict(d=128, block_l=256, G=1), 2), (dict(d=128, block_l=256, G=8), 2), (dict(block_l=512), 2),
])
def test_validation_before_any_cuda(L, kw, status):
    p = params(**kw)
    if status == 0:
        assert L.distr_attn_workspace_size(ctypes.byref(p)) > 0
        return
    rc = L.distr_attn_fwd_ex(FAKE, FAKE, FAKE, FAKE, ctypes.byref(p), None)
    assert rc == status, (rc, L.distr_attn_last_error())
    assert L.distr_attn_last_error().decode() != ""
    assert L.distr_attn_workspace_size(ctypes.byref(p)) == 0


def test_null_pointers_rejected(L):
    p = params()
    assert L.distr_attn_fwd_ex(None, FAKE, FAKE, FAKE, ctypes.byref(p), None) == 1
    assert L.distr_attn_fwd_ex(FAKE, FAKE, FAKE, FAKE, None, None) == 1
    assert L.distr_attn_hash(FAKE, ctypes.byref(p), None) == 1  # no export buffer
    assert L.distr_attn_projection(0, 64, None) == 1


def test_workspace_size_formula(L):
    # distr, bf16: only K^T [BHkv][d][N_pad] bf16 (the attention CTA hashes its own Q blocks)
    p = params(B=2, H=4, N=1000, d=128, block_l=128, G=2)
    BH, nqb, N_pad = 8, 8, 1000
    al = lambda x: (x + 255) // 256 * 256
    # ... or, when larger, the global-grouping variant: perm [BH][d] u8 + sign patterns [BH][d] u16
    # + Q̂ and K̂ [BH][N][d/G*]
    glob = al(BH * 128) + al(BH * 128 * 2) + 2 * al(BH * 1000 * 64 * 2)
    assert L.distr_attn_workspace_size(ctypes.byref(p)) == max(al(BH * 128 * N_pad * 2), glob)
    # distr, fp32: perm [BH][nqb][d] + K^T + bf16 copies of Q and V
    p = params(B=2, H=4, N=1000, d=128, block_l=128, G=2, dtype=1)
    want = al(BH * nqb * 128) + al(BH * 128 * N_pad * 2) + 2 * al(BH * 1000 * 128 * 2)
    assert L.distr_attn_workspace_size(ctypes.byref(p)) == want


def test_status_strings(L):
    for s in range(4):
        assert L.distr_attn_status_string(s).decode()
    assert L.distr_attn_status_string(99).decode() == "unknown status"


def test_backward_workspace_size_query_is_host_only(L):
    # fused path (d=128): perm [BH][nqb][d] + Q̃ [BH][N][d] bf16 + D, lse_pad [BH][N_pad128] fp32
    # (dQ̃ is folded into dQ inside the dQ̃ kernel: no fp32 dQ̃ workspace)
    p = params(B=2, H=4, N=1000, d=128, block_l=128, G=2)
    al = lambda x: (x + 255) // 256 * 256
    BH, N, d, Np = 8, 1000, 128, 1024
    want = al(BH * 8 * d) + al(BH * N * d * 2) + 2 * al(BH * Np * 4)
    assert L.distr_attn_bwd_workspace_size(ctypes.byref(p)) == want
    assert L.distr_attn_bwd_workspace_size(ctypes.byref(params(d=96))) == 0
    assert da.distr_attn_bwd_workspace_size((2, 4, 1000, 128), 4) == want


def test_binding_rejects_bad_exports_and_lse():
    import torch
    q = torch.zeros((1, 2, 100, 64), dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="lse"):
        da.make_params(q, q, block_l=64, group_size=2, lse=torch.zeros((1, 2, 99)))
    with pytest.raises(ValueError, match="lse"):
        da.make_params(q, q, block_l=64, group_size=2, lse=torch.zeros((1, 2, 100), dtype=torch.float64))
    with pytest.raises(ValueError, match="bucket_ids"):
        da.make_params(q, q, block_l=64, group_size=2, bucket_ids=torch.zeros((1, 2, 1, 64), dtype=torch.int16))
    with pytest.raises(ValueError, match="perm"):
        da.make_params(q, q, block_l=64, group_size=2, perm=torch.zeros((1, 2, 2, 64), dtype=torch.int16))
    with pytest.raises(ValueError, match="contiguous"):
        da.make_params(q, q, block_l=64, group_size=2, lse=torch.zeros((1, 100, 2)).transpose(1, 2))
    ok = da.make_params(q, q, block_l=64, group_size=2, lse=torch.zeros((1, 2, 100)),
                        bucket_ids=torch.zeros((1, 2, 2, 64), dtype=torch.int16),
                        perm=torch.zeros((1, 2, 2, 64), dtype=torch.uint8))
    assert ok.lse and ok.bucket_ids and ok.perm


def test_library_has_no_cublas_dependency(L):
    # every GEMM of the forward and backward runs in this library's tcgen05 kernels
    import subprocess
    deps = subprocess.run(["ldd", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "cublas" not in deps.lower()
    syms = subprocess.run(["nm", "-D", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "cublas" not in syms.lower()
