#!/bin/bash
# ncu launch lists of one backward call (C4-16k, d given) for the in-tree build and tools/exp variants
O=gpurun_out/bwd_ncu2; mkdir -p $O; d=${D:-32}
cp paper_2507_17245_b200/libdistr_attn.so /tmp/lib_default.so
for v in default "$@"; do
  [ $v != default ] && cp tools/exp/lib_$v.so paper_2507_17245_b200/libdistr_attn.so
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control ${CC:-none} --csv --log-file $O/launch_${v}_d$d.csv python tools/bwd_one.py 2 $d > $O/ncu_$v.log 2>&1
done
cp /tmp/lib_default.so paper_2507_17245_b200/libdistr_attn.so
