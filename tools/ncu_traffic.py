"""Write profiles/ncu_traffic.json from an `ncu --set full` raw-page CSV of the attention kernel.

    python tools/ncu_traffic.py <raw.csv> <config> <out.json> [source note]

Records dram__bytes_read.sum + dram__bytes_write.sum of the (first) attn_kernel launch in the CSV
and the sha of the kernel sources it was captured on (bench.py reports the figure as
roofline.traffic only while the sources are unchanged). Run it on the box, next to the capture.
"""
import csv, io, json, os, sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import kernel_src_sha  # noqa: E402


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return float(v.replace(",", "")) * scale


def main(raw, config, out, note=""):
    rows = list(csv.reader(io.StringIO(open(raw).read())))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        if "attn_kernel" not in name:
            continue
        rd = to_bytes(vals[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(vals[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        rec = {"source": note or f"ncu --set full, {raw}", "kernel": name, "kernel_src_sha": kernel_src_sha(),
               f"{config}_attn_bytes_per_launch": rd + wr, "read_bytes": rd, "write_bytes": wr}
        json.dump(rec, open(out, "w"), indent=1)
        print(json.dumps(rec))
        return
    raise SystemExit("no attn_kernel row in " + raw)


if __name__ == "__main__":
    main(*sys.argv[1:])
