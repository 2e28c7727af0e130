"""Small forward / backward calls for compute-sanitizer runs (racecheck, synccheck, memcheck):
one distr and one exact forward (bf16, causal, GQA, ragged N), one fp32 forward, one backward."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_17245_b200 as da
from synth import Config, make_qkv

c = Config("s", 1, 2, 1, 300, 128, 128, 2, True, "bf16", 3)
q, k, v = make_qkv(c, device="cuda")
lse = torch.empty((1, 2, 300), device="cuda")
o = da.distr_attn_fwd_ex(q, k, v, block_l=128, group_size=2, causal=True, lse=lse)
da.exact_attn_fwd_ex(q, k, v, block_l=128, causal=True)
c64 = Config("s", 1, 2, 2, 197, 64, 64, 2, False, "bf16", 4)
q2, k2, v2 = make_qkv(c64, device="cuda")
da.distr_attn_fwd_ex(q2, k2, v2, block_l=64, group_size=2)
cf = Config("s", 1, 1, 1, 200, 64, 64, 2, False, "f32", 5)
qf, kf, vf = make_qkv(cf, device="cuda")
da.distr_attn_fwd_ex(qf, kf, vf, block_l=64, group_size=2)
g = torch.Generator(device="cuda").manual_seed(1)
do = torch.randn(q.shape, generator=g, device="cuda").bfloat16()
da.distr_attn_bwd_ex(q, k, v, o, do, lse, block_l=128, group_size=2, causal=True)
# non-causal backward at d = 64 and d = 32 (the other template instances of the fused kernels)
for dd, seed in ((64, 6), (32, 7)):
    cb = Config("s", 1, 2, 2, 260, dd, 128, 2, False, "bf16", seed)
    qb, kb, vb = make_qkv(cb, device="cuda")
    lb = torch.empty((1, 2, 260), device="cuda")
    ob = da.distr_attn_fwd_ex(qb, kb, vb, block_l=128, group_size=2, lse=lb)
    da.distr_attn_bwd_ex(qb, kb, vb, ob, torch.randn(qb.shape, generator=g, device="cuda").bfloat16(), lb,
                         block_l=128, group_size=2)
torch.cuda.synchronize()
print("sanitize workload done")
