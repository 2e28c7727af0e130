O=gpurun_out/mb; mkdir -p $O
./tools/mb/ex2v > $O/ex2v.txt 2>&1
DA_PREHASH=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prep_kernel|attn_kernel" --csv --log-file $O/ph_launch.csv python tools/sweep.py --no-error --steps 1 --warmup 0 --only "C2,C4 N=4096 G*=2" > $O/ph_ncu.log 2>&1
