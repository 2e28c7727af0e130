#!/bin/bash
# A/B timing of library variants built by tools/build_variant.sh (tools/exp/lib_<name>.so):
# correctness diag, bench per EMU, clock64 trace. Usage: bash tools/gpu_ab.sh base pingpong ...
O=gpurun_out; mkdir -p $O
cp paper_2507_17245_b200/libdistr_attn.so tools/exp/lib_intree.so
for v in "$@"; do
  cp tools/exp/lib_$v.so paper_2507_17245_b200/libdistr_attn.so
  timeout -s KILL 90 python tools/diag.py exact distr > $O/diag_$v.log 2>&1 || echo "diag failed rc=$?" >> $O/diag_$v.log
  grep -q "failed" $O/diag_$v.log && continue
  for e in ${EMUS:-0 2}; do
    DA_EMU=$e timeout -s KILL 120 python bench.py --steps 5 --no-e2e --no-cpu --no-parity > $O/bench_${v}_e$e.log 2>&1
  done
  [ -n "$SWEEP" ] && timeout -s KILL 300 python tools/sweep.py --only "$SWEEP" > $O/sweep_$v.json 2>&1
  timeout -s KILL 60 python tools/trace.py distr > $O/trace_${v}_distr.log 2>&1
  timeout -s KILL 60 python tools/trace.py exact > $O/trace_${v}_exact.log 2>&1
done
cp tools/exp/lib_intree.so paper_2507_17245_b200/libdistr_attn.so
