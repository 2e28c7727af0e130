"""Backward timing (distr_attn_bwd_ex): CUDA events around the C call, after
warm-up (median of 7 batches), on the C4 shape (B=1 H=16) at N in {4k, 16k}, G* in {1, 2}, for the fused tcgen05
kernels (d = 32, 64, 128; G* = 1, 2).

    python tools/bench_bwd.py > gpurun_out/bwd.json

Algorithmic FLOP per call: five GEMMs of 2·N·N_k·d (Ŝ = Q̃Kᵀ, dP = dO Vᵀ, dV = Pᵀ dO, dQ̃ = dŜ K,
dK = dŜᵀ Q̃) per head ("tflops_executed" counts these; the fused path runs seven MMAs per tile
pair — Ŝ and dP in both of its kernels — so its tensor pipe does 7/5 of that). Roofline against
MEASURED_PEAKS bf16.
"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2507_17245_b200 as da
from synth import CONFIGS, make_qkv

peaks = {}
try:
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
except Exception:
    pass
peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 2250.0))
for N in (4096, 16384):
  for d in (32, 64, 128):
    path = "fused"
    for G in (1, 2):
        c = CONFIGS["C4"].with_(B=1, H=16, H_kv=16, N=N, d=d, group_size=G)
        q, k, v = make_qkv(c, device="cuda")
        dout = torch.randn_like(q.float()).bfloat16()
        lse = torch.empty(q.shape[:3], dtype=torch.float32, device="cuda")
        out = da.distr_attn_fwd_ex(q, k, v, group_size=G, lse=lse)
        for _ in range(2):
            da.distr_attn_bwd_ex(q, k, v, out, dout, lse, group_size=G)
        # median of 7 timed batches of 5 calls: long d = 128 runs sit at the 1 kW power cap and
        # their clock (hence time) moves by several percent between batches
        steps, times = 5, []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(steps):
                da.distr_attn_bwd_ex(q, k, v, out, dout, lse, group_size=G)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / steps)
        times.sort()
        ms = times[len(times) // 2]
        flop = 5 * 2.0 * N * N * c.d * c.H
        rec = {"path": path, "N": N, "G": G, "B": 1, "H": 16, "d": d, "bwd_ms": ms,
               "bwd_ms_min": times[0], "bwd_ms_max": times[-1],
               "tflops_executed": flop / (ms * 1e-3) / 1e12, "peak_tflops": peak,
               "frac_of_peak": flop / (ms * 1e-3) / 1e12 / peak}
        print(json.dumps(rec), flush=True)
