#!/bin/bash
# Forward A/B (in-tree build vs tools/exp variants, alternating): quick parity, CTA timelines, C5 bench.
O=gpurun_out/fwd_ab3; mkdir -p $O
cp paper_2507_17245_b200/libdistr_attn.so /tmp/lib_default.so
use() { if [ $1 = default ]; then cp /tmp/lib_default.so paper_2507_17245_b200/libdistr_attn.so; else cp tools/exp/lib_$1.so paper_2507_17245_b200/libdistr_attn.so; fi; }
for v in "$@"; do
  use $v
  timeout -s KILL 180 python tools/quick.py > $O/quick_$v.log 2>&1; echo "rc=$?" >> $O/quick_$v.log
  timeout -s KILL 60 python tools/trace.py distr > $O/trace_distr_$v.log 2>&1
done
for rep in 1 2; do
  for v in default "$@"; do
    use $v
    timeout -s KILL 600 python bench.py --no-e2e --no-cpu --no-parity --steps 10 > $O/bench_${v}_$rep.log 2>&1
  done
done
use default
