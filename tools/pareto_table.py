"""Markdown table of a Pareto sweep (tools/pareto.py output): python tools/pareto_table.py pareto.json"""
import json, sys
print("| d | grouping | G* | S width | rel. error vs exact: N(0,1) / clustered / block-clustered | mean-abs (N(0,1)) "
      "| C4-16k distr ms | exact ms | speed-up |")
print("|---|---|---|---|---|---|---|---|---|")
for line in open(sys.argv[1]):
    if not line.startswith("{"):
        continue
    r = json.loads(line)
    grp = "global" if r["block_l"] == "global" else f"block l={r['block_l']}"
    e = [r[f"err_{k}"]["rel_fro"] for k in ("normal", "clustered", "block_clustered")]
    print(f"| {r['d']} | {grp} | {r['G']} | {r['DR']} | {e[0]:.3f} / {e[1]:.3f} / {e[2]:.3f} | "
          f"{r['err_normal']['mean_abs']:.4f} | {r['distr_ms']:.3f} | {r['exact_ms']:.3f} | {r['speedup_vs_exact']:.3f} |")
