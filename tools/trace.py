"""Pipeline timeline of CTA (0,0): python tools/trace.py [distr|exact] [N] [d] [block_l] [G] [causal] [H] [H_kv]
(defaults: N=16384 d=128 block_l=128 G=2 non-causal H=H_kv=16, B=1)"""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2507_17245_b200 as da
from paper_2507_17245_b200 import _native
from synth import Config, make_qkv
mode = sys.argv[1] if len(sys.argv) > 1 else "distr"
arg = lambda i, dflt: int(sys.argv[i]) if len(sys.argv) > i else dflt
N, d, L, G, causal, H = arg(2, 16384), arg(3, 128), arg(4, 128), arg(5, 2), bool(arg(6, 0)), arg(7, 16)
Hkv = arg(8, H)
c = Config("t", 1, H, Hkv, N, d, L, G, causal, "bf16", 5)
q, k, v = make_qkv(c, device="cuda")
f = ((lambda: da.distr_attn_fwd_ex(q, k, v, block_l=L, group_size=G, causal=causal)) if mode == "distr"
     else (lambda: da.exact_attn_fwd_ex(q, k, v, block_l=L, causal=causal)))
for _ in range(3): f()
buf = torch.zeros(20 * 256, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
_native.lib().distr_attn_set_trace(ctypes.c_void_p(buf.data_ptr()))
f(); torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(20, 256).astype(np.int64)
t0 = t[t > 0].min()
names = {0: "sm0 S ready", 1: "sm0 max done", 2: "sm0 P arrive", 3: "sm1 S ready", 4: "sm1 max done", 5: "sm1 P arrive",
         6: "mma S0 issued", 7: "mma S1 issued", 8: "mma P0 seen", 9: "mma P1 seen", 10: "fus K ready", 11: "fus K0 done", 12: "fus K1 done",
         13: "sm0 wait start", 14: "sm1 wait start"}
nt = int((t[2] > 0).sum())  # key tiles recorded (<= 256)
pro = t[15, :5]
if pro[0] > 0:
    print("prologue (cycles from start): proj loaded+Q landed", pro[1]-pro[0], " hash", pro[2]-pro[1], " rank", pro[3]-pro[2], " qhat", pro[4]-pro[3], " total", pro[4]-pro[0])
    print("first S0 ready after prologue end:", t[0, 0] - pro[4])
for i in list(range(0, 6)) + list(range(max(6, nt - 4), nt)):
    print(f"--- tile {i}")
    ev = sorted([(t[s, i] - t0, n) for s, n in names.items() if t[s, i] > 0])
    for c_, n in ev: print(f"  {c_:9d}  {n}")
# steady-state per-iteration stats
LO, HI = min(20, nt // 4), min(100, nt - 1)
def d(a, b, lo=LO, hi=HI): return np.median(t[b, lo:hi] - t[a, lo:hi])
print(f"median cycles (tiles {LO}..{HI}):")
print("  sm0: wait S   ", d(13, 0), " S->max", d(0, 1), " max->P", d(1, 2), " period", np.median(np.diff(t[2, LO:HI])))
print("  sm1: wait S   ", d(14, 3), " S->max", d(3, 4), " max->P", d(4, 5), " period", np.median(np.diff(t[5, LO:HI])))
print("  sm0 max->expdone", d(1, 16), " expdone->arrive", d(16, 2))
print("  P0 arrive -> mma sees", d(2, 8), " P1:", d(5, 9))
print("  mma S0 issued -> sm0 S ready (next tile)", np.median(t[0, LO + 1:HI + 1] - t[6, LO + 1:HI + 1]))
print("  fusion K ready->K0 done", d(10, 11), " K0->K1", d(11, 12), " fusion period", np.median(np.diff(t[10, LO:HI])))
