"""First-contact GPU diagnostics: each step prints as it completes (run under `timeout`)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2507_17245_b200 as da
import oracle
from synth import Config, make_qkv
from gpu_util import oracle_items, gather_items, valid_rows_mask, errors

def P(*a):
    print(*a, flush=True)

def cfg(**kw):
    base = dict(name="t", B=1, H=1, H_kv=1, N=128, d=128, block_l=128, group_size=2, causal=False, dtype="bf16", data_seed=5)
    base.update(kw); return Config(**base)

steps = sys.argv[1:] or ["hash", "exact", "distr"]
if "hash" in steps:
    c = cfg(N=300)
    q, _, _ = make_qkv(c, device="cuda")
    bk, pm = da.distr_attn_hash(q, block_l=128, group_size=2, seed=11)
    torch.cuda.synchronize()
    ob, op = oracle.hash_all(q.float().cpu().numpy(), 128, 11)
    P("hash equal:", np.array_equal(bk.cpu().numpy().view(np.uint16), ob), "perm equal:", np.array_equal(pm.cpu().numpy(), op))

def attn(c, exact, dist="normal"):
    q, k, v = make_qkv(c, device="cuda", dist=dist)
    t = time.time()
    if exact:
        out = da.exact_attn_fwd_ex(q, k, v, block_l=c.block_l, causal=c.causal)
    else:
        out = da.distr_attn_fwd_ex(q, k, v, block_l=c.block_l, group_size=c.group_size, causal=c.causal)
    torch.cuda.synchronize()
    items = [(bh, qb) for bh in range(c.B * c.H) for qb in range(c.nqb)]
    want = oracle_items(q, k, v, items, block_l=c.block_l, G=0 if exact else c.group_size, causal=c.causal)
    got = gather_items(out, items, c.block_l)
    m = valid_rows_mask(items, c.N, c.block_l, c.d)
    mx, mean = errors(got, want, m)
    P(("exact" if exact else "distr"), c.N, c.d, c.block_l, c.group_size, "causal" if c.causal else "", "max %.3e mean %.3e" % (mx, mean), "%.1f ms" % ((time.time()-t)*1e3))
    if mx > 2e-2:
        d = np.abs(got - want) * m
        r = np.argwhere(d > 2e-2)
        P("  bad elems:", len(r), "first:", r[:8].tolist())
        P("  got[0,0,:8]", got[0, 0, :8].round(4).tolist())
        P("  want[0,0,:8]", want[0, 0, :8].round(4).tolist())
        P("  row err profile:", d.max(axis=2)[0, ::16].round(3).tolist())
    return mx

if "exact" in steps:
    for N in (128, 256, 300):
        for d in (128, 64):
            attn(cfg(N=N, d=d), True)
    attn(cfg(N=300, causal=True), True)
if "distr" in steps:
    for N in (128, 300):
        for (d, l, G) in ((128, 128, 2), (128, 128, 1), (64, 128, 2), (64, 64, 2), (128, 128, 4), (128, 64, 2)):
            attn(cfg(N=N, d=d, block_l=l, group_size=G), False)
    attn(cfg(N=300, causal=True, H=4, H_kv=2), False)
P("done")
