"""Run one attention config: python tools/diag1.py N d l G causal exact"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_17245_b200 as da
from synth import Config, make_qkv
N, d, l, G, causal, exact = (int(x) for x in sys.argv[1:7])
c = Config("t", 1, 1, 1, N, d, l, G, bool(causal), "bf16", 5)
q, k, v = make_qkv(c, device="cuda")
if exact:
    out = da.exact_attn_fwd_ex(q, k, v, block_l=l, causal=bool(causal))
else:
    out = da.distr_attn_fwd_ex(q, k, v, block_l=l, group_size=G, causal=bool(causal))
torch.cuda.synchronize()
print("ok", N, d, l, G, causal, exact, torch.isfinite(out).all().item(), flush=True)
