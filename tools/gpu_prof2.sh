#!/bin/bash
# Round-2 profile pass: ncu launch list of the bench command, ncu --set full of the C5 distr and
# exact attention kernels and of the K^T prep kernel (raw + details CSV, traffic json), and
# compute-sanitizer racecheck / synccheck / memcheck over a small workload.
O=gpurun_out/${TAG:-prof2}; mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prep_kernel|attn_kernel|convert_kernel" -c 60 --csv --log-file $O/ncu_launches.csv $B > $O/ncu_launches.log 2>&1
B1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 3 -c 1 -o $O/prof_distr -f $B1 > $O/ncu_distr.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 7 -c 1 -o $O/prof_exact -f $B1 > $O/ncu_exact.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:prep_kernel -s 3 -c 1 -o $O/prof_prep -f $B1 > $O/ncu_prep.log 2>&1
for k in distr exact prep; do
  ncu -i $O/prof_$k.ncu-rep --page raw --csv > $O/raw_$k.csv 2>&1
  ncu -i $O/prof_$k.ncu-rep --page details --csv > $O/details_$k.csv 2>&1
  [ $k != prep ] && ncu -i $O/prof_$k.ncu-rep --page source --csv --print-source sass > $O/sass_$k.csv 2>&1
  python tools/ncu_summary.py $O/prof_$k.ncu-rep $O/ncu_$k > /dev/null 2>&1
done
python tools/ncu_traffic.py $O/raw_distr.csv C5 $O/ncu_traffic.json "ncu --set full of attn_kernel<128,distr,G=2,HB=1,EMU=2> on C5 (B=32,H=32,N=16k,d=128), $TAG" > $O/ncu_traffic.log 2>&1
rm -f $O/*.ncu-rep
for tool in racecheck synccheck memcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > $O/sanitize_$tool.log 2>&1; echo "rc=$?" >> $O/sanitize_$tool.log
done
ls -la $O
