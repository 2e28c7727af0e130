"""Summarise an ncu source-page SASS CSV (tools/gpu_prof.sh): stall samples per instruction class
inside an address window, and the hottest instructions. Usage: sass_stalls.py file.csv [lo hi]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
def num(x):
    try: return float(x)
    except: return 0.0
tot = collections.Counter(); by_op = collections.Counter(); samples = 0
ins = []
for r in data:
    if len(r) < len(hdr): continue
    s = int(num(r[ix["Warp Stall Sampling (All Samples)"]]))
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"): op = r[ix["Source"]].split()[1]
    samples += s
    by_op[op.split(".")[0]] += s
    for h in stall_cols: tot[h] += num(r[ix[h]])
    ins.append((s, r[ix["Address"]][-5:], r[ix["Source"]].strip()[:60], {h[6:]: int(num(r[ix[h]])) for h in stall_cols if num(r[ix[h]]) > 0.1 * max(1, s)}))
print("total samples", samples)
print("stall reasons:", ", ".join(f"{k[6:]} {v/samples*100:.1f}%" for k, v in tot.most_common(12)))
print("samples by opcode:", ", ".join(f"{k} {v/samples*100:.1f}%" for k, v in by_op.most_common(15)))
exc = [(num(r[ix["L1 Wavefronts Shared Excessive"]]), num(r[ix["L1 Wavefronts Shared"]]), r[ix["Address"]][-5:],
        r[ix["Source"]].strip()[:60]) for r in data if len(r) >= len(hdr) and "L1 Wavefronts Shared Excessive" in ix]
tw = sum(e[1] for e in exc); te = sum(e[0] for e in exc)
if tw:
    print(f"shared wavefronts {tw:.3e}, excessive (bank conflicts) {te:.3e} = {te / tw * 100:.1f}%; top excessive:")
    for e, w, a, src in sorted(exc, reverse=True)[:12]:
        if e > 0: print(f"  {e / te * 100:5.1f}% of excessive  {a} {src}  (wavefronts {w:.2e})")
print("hottest instructions:")
for s, a, src, st in sorted(ins, reverse=True)[:40]:
    print(f"  {s/samples*100:5.2f}% {a} {src:60s} {st}")
