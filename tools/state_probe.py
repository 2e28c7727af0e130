"""Does the library's state change DistrAttention's speed? Times d=128 block_l=128 G*=2 at the C4
16k shape fresh, then after calls of other variants (block_l 64 / 256, G* 4 / 8, the global
variant, the exact kernel, a small N=4096 H=8 shape), each time 10 calls after 3."""
import os, sys, json
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


c = CONFIGS["C4"].with_(B=1, H=16, H_kv=16, N=16384, d=128, block_l=128, group_size=2)
q, k, v = make_qkv(c, device="cuda")
out = torch.empty_like(q)
mode = sys.argv[1] if len(sys.argv) > 1 else "scratch"
if mode == "workspace":  # caller workspace: one torch allocation, reused by every call
    ws = torch.empty(da.distr_attn_workspace_size(q.shape, 128, 2, h_kv=16) if False else 1 << 28, dtype=torch.uint8,
                     device="cuda")
    base = lambda: da.distr_attn_fwd_ex(q, k, v, out, block_l=128, group_size=2, workspace=ws)
else:
    base = lambda: da.distr_attn_fwd_ex(q, k, v, out, block_l=128, group_size=2)
print(json.dumps({"state": "fresh", "mode": mode, "ms": t(base)}), flush=True)
small = CONFIGS["C4"].with_(B=1, H=8, H_kv=8, N=4096, d=128, block_l=128, group_size=2)
qs, ks, vs = make_qkv(small, device="cuda")
others = [("exact", lambda: da.exact_attn_fwd_ex(q, k, v, out)),
          ("small N=4096 H=8", lambda: da.distr_attn_fwd_ex(qs, ks, vs, block_l=128, group_size=2)),
          ("block_l=64", lambda: da.distr_attn_fwd_ex(q, k, v, out, block_l=64, group_size=4)),
          ("block_l=256", lambda: da.distr_attn_fwd_ex(q, k, v, out, block_l=256, group_size=2)),
          ("G*=8", lambda: da.distr_attn_fwd_ex(q, k, v, out, block_l=128, group_size=8)),
          ("global", lambda: da.distr_attn_global_fwd_ex(q, k, v, out, group_size=2))]
for name, fn in others:
    o = t(fn, 3)
    print(json.dumps({"state": f"after {name}", "other_ms": o, "ms": t(base)}), flush=True)
print(json.dumps({"state": "again", "ms": t(base)}), flush=True)
