"""Fit the planner's cost model (api.cu kDistrCost / kExact*) to measured sweeps.

    python tools/fit_planner.py profiles/r02_v2/sweep.json profiles/r02_v2/sweep_l256.json

Model per kernel variant: t_us * f = waves * (prologue + steps * step) (+ the K^T pass and launch
overheads, added separately in the planner), waves = ceil(CTAs / 148) for non-causal jobs
(all CTAs equal), CTAs = B*H*ceil(nqt/2). Least squares over the C4 N sweep (d = 128); d = 64
variants are scaled from the d = 128 fit by the CTA-timeline ratios of tools/calibrate.sh.
"""
import json, math, sys
import numpy as np

F_MHZ = 1800.0
rows = [json.loads(l) for f in sys.argv[1:] for l in open(f)]


def waves_and_steps(r):
    nqt = -(-r["N"] // 128)
    ctas = r["B"] * r["H"] * -(-nqt // 2)
    return math.ceil(ctas / 148), nqt


def fit(points):
    """Non-negative least squares on RELATIVE residuals (every N counts the same)."""
    from scipy.optimize import nnls
    A = np.array([[w / t, w * s / t] for w, s, t in points], float)
    (pro, step), _ = nnls(A, np.ones(len(points)))
    return pro, step


var = {}
for r in rows:
    if not r["case"].startswith("C4"):
        continue
    w, s = waves_and_steps(r)
    kt_us = 4.0 + 4.0 * r["B"] * r["H_kv"] * r["N"] * r["d"] / 5.1e6
    var.setdefault(("distr", r["block_l"], r["G"]), []).append((w, s, (r["distr_ms"] * 1e3 - 4.0 - kt_us) * F_MHZ))
    var.setdefault(("exact", 0, 1), []).append((w, s, (r["exact_ms"] * 1e3 - 4.0) * F_MHZ))
for k, pts in sorted(var.items()):
    pro, step = fit(pts)
    print(k, f"prologue {pro:.0f} clk, step {step:.0f} clk", "residuals %:",
          [round((w * (pro + s * step) - t) / t * 100, 1) for w, s, t in pts])
