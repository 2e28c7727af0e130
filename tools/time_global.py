"""Timing of the global-grouping variant (distr_attn_global_fwd_ex) against the block-wise
forward and the exact kernel on the C4 shape (B=1 H=16 d=128), CUDA events, 10 calls after 3."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_17245_b200 as da
from synth import CONFIGS, make_qkv


def t(fn, steps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


for N in (4096, 16384, 65536):
    for G in (2, 4):
        c = CONFIGS["C4"].with_(N=N, group_size=G)
        q, k, v = make_qkv(c, device="cuda")
        rec = {"N": N, "G": G,
               "global_ms": t(lambda: da.distr_attn_global_fwd_ex(q, k, v, group_size=G)),
               "blockwise_ms": t(lambda: da.distr_attn_fwd_ex(q, k, v, block_l=128, group_size=G)),
               "exact_ms": t(lambda: da.exact_attn_fwd_ex(q, k, v))}
        print(json.dumps(rec), flush=True)
