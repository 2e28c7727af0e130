"""Summarise an ncu report into text files that can be committed under profiles/.

    python tools/ncu_summary.py gpurun_out/prof_attn.ncu-rep profiles/r01_v5/ncu_attn

writes <prefix>_details.csv (ncu --page details) and <prefix>_raw_selected.txt (the metrics the
roofline / DESIGN.md cite: time, DRAM bytes, tensor/XU/FMA/ALU pipes, shared-memory traffic).
"""
import csv, io, subprocess, sys

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpc__cycles_elapsed.max",
        "sm__pipe_tensor_cycles_active", "sm__inst_executed_pipe_xu", "sm__pipe_fma_cycles_active",
        "sm__pipe_fmaheavy_cycles_active", "sm__pipe_alu_cycles_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared",
        "l1tex__data_pipe_tc_wavefronts_mem_shared", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_bank_reads", "l1tex__data_bank_writes", "l1tex__throughput", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "sm__throughput",
        "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum", "smsp__mem_tensor_writes_op_utcmma.sum",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum", "dram__throughput",
        "gpu__dram_throughput")


def main(rep, prefix):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    open(prefix + "_details.csv", "w").write(det)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = [f"kernel: {vals[hdr.index('Kernel Name')]}"]
    for h, u, v in zip(hdr, units, vals):
        if any(h.startswith(k) for k in KEYS) and ("pct" in h or h.endswith((".sum", ".max", ".avg", "_size", "thread"))
                                                   or h.endswith("per_second")):
            if "peak_sustained." in h or h.endswith(".peak_sustained"):
                continue
            out.append(f"{h} | {u} | {v}")
    open(prefix + "_raw_selected.txt", "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
