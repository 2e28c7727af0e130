O=gpurun_out; mkdir -p $O
B="python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity"
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:prep_kernel -s 3 -c 1 -o $O/prof_prep -f $B > $O/ncu1.log 2>&1
