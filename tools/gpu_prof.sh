#!/bin/bash
# ncu --set full (with source) of the distr and exact attention kernels at C4 N=16k; exports the
# raw and per-instruction (source page, SASS) CSVs and drops the .ncu-rep files (too large to ship).
O=gpurun_out; mkdir -p $O
B="python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 3 -c 1 -o $O/prof_distr -f $B > $O/ncu1.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 7 -c 1 -o $O/prof_exact -f $B > $O/ncu2.log 2>&1
for k in distr exact; do
  ncu -i $O/prof_$k.ncu-rep --page raw --csv > $O/raw_$k.csv 2>&1
  ncu -i $O/prof_$k.ncu-rep --page source --csv --print-source sass > $O/sass_$k.csv 2>&1
  ncu -i $O/prof_$k.ncu-rep --page details --csv > $O/details_$k.csv 2>&1
  rm -f $O/prof_$k.ncu-rep
done
ls -la $O
