import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2507_17245_b200 as da
from synth import CONFIGS, make_qkv
G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
D = int(sys.argv[2]) if len(sys.argv) > 2 else 128
c = CONFIGS["C4"].with_(B=1, H=16, H_kv=16, N=16384, d=D, group_size=G)
q, k, v = make_qkv(c, device="cuda")
dout = torch.randn_like(q.float()).bfloat16()
lse = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
out = da.distr_attn_fwd_ex(q, k, v, group_size=G, lse=lse)
for _ in range(3):
    da.distr_attn_bwd_ex(q, k, v, out, dout, lse, group_size=G)
torch.cuda.synchronize()
