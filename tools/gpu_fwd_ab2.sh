#!/bin/bash
# Forward A/B of build variants x exact-kernel EMU (the exact reference must run at its best
# setting): quick parity + CTA timelines per variant, then alternating C5 benches (kernel-only).
O=gpurun_out/fwd_ab2; mkdir -p $O
cp paper_2507_17245_b200/libdistr_attn.so /tmp/lib_default.so
use() { if [ $1 = default ]; then cp /tmp/lib_default.so paper_2507_17245_b200/libdistr_attn.so; else cp tools/exp/lib_$1.so paper_2507_17245_b200/libdistr_attn.so; fi; }
for v in "$@"; do
  use $v
  timeout -s KILL 180 python tools/quick.py > $O/quick_$v.log 2>&1; echo "rc=$?" >> $O/quick_$v.log
  timeout -s KILL 60 python tools/trace.py distr > $O/trace_distr_$v.log 2>&1
  DA_EMU_EXACT=2 timeout -s KILL 60 python tools/trace.py exact > $O/trace_exact_$v.log 2>&1
done
for rep in 1 2; do
  for v in "$@"; do
    use $v
    for ee in 0 2; do
      DA_EMU_EXACT=$ee timeout -s KILL 600 python bench.py --no-e2e --no-cpu --no-parity --steps 10 > $O/bench_${v}_e${ee}_$rep.log 2>&1
    done
    DA_EMU_EXACT=2 timeout -s KILL 300 python tools/sweep.py --no-error --only "C4 N=16384,C4 N=32768 G*=2" > $O/sweep_${v}_$rep.json 2>&1
  done
done
use default
