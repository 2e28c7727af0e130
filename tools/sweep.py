"""Per-config timings (distr vs own exact kernel) for every BASELINE.json config + the C4 N sweep.

    python tools/sweep.py [--steps K] > gpurun_out/sweep.json   (one JSON line per case)

Call times: CUDA events around 10 back-to-back calls (no per-call events, so the K^T pass and
the attention kernel may overlap); kernel times from a second pass with events recorded around
the launches inside the C call (distr_attn_set_profile_events). Each row also carries, on sampled
Q blocks, the GPU output against the oracle's DistrAttention (parity) and against the exact-
attention oracle (max-abs, mean-abs, relative Frobenius error: SURVEY §8(c) item 8), and with
--plan the planner's pick measured. Inputs are regenerated per case on the device.
"""
import argparse, ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2507_17245_b200 as da
from paper_2507_17245_b200 import _native
from synth import CONFIGS, C4_SWEEP_N, make_qkv

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--only", default="", help="comma-separated case-name prefixes (default: all)")
ap.add_argument("--block-l", type=int, default=0, help="override block_l of every case (e.g. 256)")
ap.add_argument("--no-error", action="store_true", help="skip the sampled oracle comparisons")
ap.add_argument("--plan", action="store_true",
                help="also run distr_attn_choose's pick for each case (max_group_size = the case's G*)")
args = ap.parse_args()
L = _native.lib()
cases = [("C1", CONFIGS["C1"]), ("C2", CONFIGS["C2"]), ("C3", CONFIGS["C3"])]
cases += [(f"C4 N={n} G*={g}", CONFIGS["C4"].with_(N=n, group_size=g)) for n in C4_SWEEP_N for g in (2, 4)]
cases += [("C5 1-GPU", CONFIGS["C5"])]
if args.only:
    cases = [c for c in cases if any(c[0].startswith(p) for p in args.only.split(","))]
if args.block_l:
    cases = [(f"{n} l={args.block_l}", c.with_(block_l=args.block_l)) for n, c in cases]


def timed(fn):
    """(ms per call over `steps` back-to-back calls, attention-kernel ms). The call time is taken
    with no per-call events armed (the K^T pass and the attention kernel may overlap through
    programmatic dependent launch); the kernel split comes from a second pass with the events
    recorded between the launches (which serialises them)."""
    for _ in range(args.warmup):
        fn(None)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        fn(None)
    t1.record()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    for e3 in evs:
        for e in e3:
            e.record()
    torch.cuda.synchronize()
    for e3 in evs:
        fn(e3)
    torch.cuda.synchronize()
    attn = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    return t0.elapsed_time(t1) / args.steps, attn


for name, c in cases:
    q, k, v = make_qkv(c, device="cuda")
    out = torch.empty_like(q)

    def run(evs, exact=False):
        if evs is not None:
            L.distr_attn_set_profile_events(*[ctypes.c_void_p(e.cuda_event) for e in evs])
        if exact:
            da.exact_attn_fwd_ex(q, k, v, out, block_l=c.block_l, causal=c.causal)
        else:
            da.distr_attn_fwd_ex(q, k, v, out, block_l=c.block_l, group_size=c.group_size, causal=c.causal)

    d_ms, d_attn = timed(lambda e: run(e))
    x_ms, x_attn = timed(lambda e: run(e, True))
    pairs = c.B * c.H * c.N * c.N * (0.5 if c.causal else 1.0)
    DR = max(1, 128 // c.block_l) * c.d // c.group_size
    rec = {"case": name, "B": c.B, "H": c.H, "H_kv": c.H_kv, "N": c.N, "d": c.d, "block_l": c.block_l,
           "G": c.group_size, "causal": c.causal, "dtype": c.dtype,
           "distr_ms": d_ms, "distr_attn_kernel_ms": d_attn, "exact_ms": x_ms, "exact_attn_kernel_ms": x_attn,
           "speedup": x_ms / d_ms,
           "distr_tflops_executed": pairs * (2 * DR + 2 * c.d) / (d_attn * 1e-3) / 1e12,
           "exact_tflops": pairs * 4 * c.d / (x_attn * 1e-3) / 1e12,
           "full_d_equiv_tflops": pairs * 4 * c.d / (d_ms * 1e-3) / 1e12}
    if not args.no_error:
        # sampled Q blocks (first, last, one random, of two heads): the GPU DistrAttention output
        # against the oracle's DistrAttention (parity, the north-star tolerance) and against the
        # exact-attention oracle (the approximation error the config reports)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from gpu_util import errors, gather_items, oracle_items, valid_rows_mask
        from synth import sample_items
        run(None)
        torch.cuda.synchronize()
        items = sample_items(c, n_heads=2, per_head=3)
        got = gather_items(out, items, c.block_l)
        mask = valid_rows_mask(items, c.N, c.block_l, c.d)
        want = oracle_items(q, k, v, items, block_l=c.block_l, G=c.group_size, causal=c.causal)
        ex = oracle_items(q, k, v, items, block_l=c.block_l, G=0, causal=c.causal)
        pmx, pmean = errors(got, want, mask)
        emx, emean = errors(got, ex, mask)
        dg, de = (got - ex)[mask], ex[mask]
        rec["parity_vs_oracle"] = {"max_abs": pmx, "mean_abs": pmean, "items": len(items),
                                   "ok": bool(pmx <= 2e-2 and pmean <= 2e-3)}
        rec["error_vs_exact"] = {"max_abs": emx, "mean_abs": emean,
                                 "rel_fro": float(np.linalg.norm(dg) / np.linalg.norm(de))}
    if args.plan:
        ch = da.distr_attn_choose(c.B, c.H, c.H_kv, c.N, c.d, causal=c.causal, max_group_size=c.group_size)
        if ch["distr"]:
            def run_plan(evs):
                if evs is not None:
                    L.distr_attn_set_profile_events(*[ctypes.c_void_p(e.cuda_event) for e in evs])
                da.distr_attn_fwd_ex(q, k, v, out, block_l=ch["block_l"], group_size=ch["group_size"],
                                     causal=c.causal)
            p_ms, _ = timed(run_plan)
        else:
            p_ms = x_ms
        rec["plan"] = dict(ch, measured_ms=p_ms)
    print(json.dumps(rec), flush=True)
    del q, k, v, out
    torch.cuda.empty_cache()
