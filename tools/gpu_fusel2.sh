O=gpurun_out/nofuse; mkdir -p $O
cp tools/exp/lib_fusel2.so /tmp/l.so; cp paper_2507_17245_b200/libdistr_attn.so /tmp/d.so
cp /tmp/l.so paper_2507_17245_b200/libdistr_attn.so; timeout -s KILL 180 python tools/quick.py > $O/quick_fusel2.log 2>&1; echo "rc=$?" >> $O/quick_fusel2.log
cp /tmp/d.so paper_2507_17245_b200/libdistr_attn.so
VARS=fusel2 bash tools/gpu_nofuse.sh
