#!/bin/bash
# Planner calibration: CTA-0 timelines (steady period per key tile, prologue) for the kernel
# variants the planner chooses between. Output: gpurun_out/$TAG/calib.txt
O=gpurun_out/${TAG:-calib}; mkdir -p $O; : > $O/calib.txt
for d in 64 128; do
  echo "exact d=$d" >> $O/calib.txt
  timeout -s KILL 60 python tools/trace.py exact 16384 $d 128 1 0 16 16 | tail -7 >> $O/calib.txt 2>&1
  for lg in "128 2" "128 4" "256 2" "256 4" "64 2"; do
    set -- $lg
    echo "distr d=$d l=$1 G=$2" >> $O/calib.txt
    timeout -s KILL 60 python tools/trace.py distr 16384 $d $1 $2 0 16 16 2>&1 | grep -E "prologue|period|wait S" >> $O/calib.txt
  done
done
