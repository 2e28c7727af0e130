"""Fast first-contact check of a new kernel build (run under `timeout`): a few small shapes of
the distr and exact kernels against the CPU oracle, printing max/mean abs error per case."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2507_17245_b200 as da
from gpu_util import oracle_items, gather_items, valid_rows_mask, errors
from synth import Config, make_qkv

cases = [  # name, N, d, l, G, causal, H, Hkv
    ("d128 N=300", 300, 128, 128, 2, False, 2, 2), ("d128 N=1000 causal", 1000, 128, 128, 2, True, 2, 1),
    ("d64 l=64 N=197", 197, 64, 64, 2, False, 2, 2), ("d128 l=256 G4 N=700", 700, 128, 256, 4, False, 2, 2),
    ("d32 N=333 causal", 333, 32, 128, 2, True, 2, 2), ("d128 N=2048", 2048, 128, 128, 2, False, 1, 1)]
ok = True
for name, N, d, l, G, causal, H, Hkv in cases:
    c = Config("q", 1, H, Hkv, N, d, l, G, causal, "bf16", 3)
    q, k, v = make_qkv(c, device="cuda")
    items = [(bh, qb) for bh in range(H) for qb in range(c.nqb)]
    for exact in (False, True):
        out = (da.exact_attn_fwd_ex(q, k, v, block_l=l, causal=causal) if exact else
               da.distr_attn_fwd_ex(q, k, v, block_l=l, group_size=G, causal=causal))
        torch.cuda.synchronize()
        want = oracle_items(q, k, v, items, block_l=l, G=0 if exact else G, causal=causal)
        mx, mean = errors(gather_items(out, items, l), want, valid_rows_mask(items, N, l, d))
        good = mx <= 2e-2 and mean <= 2e-3
        ok &= good
        print(f"{'exact' if exact else 'distr'} {name}: max {mx:.2e} mean {mean:.2e} {'ok' if good else 'FAIL'}", flush=True)
print("QUICK", "PASS" if ok else "FAIL")
sys.exit(0 if ok else 1)
