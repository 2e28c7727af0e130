#!/bin/bash
# Round-2 final evidence (session 3): the round-2 pass (tests, smoke, bench, sweeps, backward
# timings, traces, ncu, sanitizers) plus ncu of the backward kernels (launch list at running and at
# base clock, --set full of the dK/dV and dQ̃ kernels at C4-16k d=128 G*=2).
O=gpurun_out/${TAG:-r3}; mkdir -p $O
TAG=${TAG:-r3} bash tools/gpu_round2.sh > /dev/null 2>&1
for cc in none base; do
  timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control $cc --csv --log-file $O/ncu_bwd_launches_$cc.csv python tools/bwd_one.py 2 128 > /dev/null 2>&1
done
for kn in bwd_kv_kernel bwd_q_kernel; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$kn -s 1 -c 1 -o $O/prof_$kn -f python tools/bwd_one.py 2 128 > $O/ncu_$kn.log 2>&1
  ncu -i $O/prof_$kn.ncu-rep --page raw --csv > $O/raw_$kn.csv 2>&1
  python tools/ncu_summary.py $O/prof_$kn.ncu-rep $O/ncu_$kn > /dev/null 2>&1
  rm -f $O/prof_$kn.ncu-rep
done
ls -la $O
