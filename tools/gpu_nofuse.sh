O=gpurun_out/nofuse; mkdir -p $O
cp paper_2507_17245_b200/libdistr_attn.so /tmp/lib_default.so
for rep in 1 2; do
 for v in default ${VARS:-nofuse}; do
  if [ $v = default ]; then cp /tmp/lib_default.so paper_2507_17245_b200/libdistr_attn.so; else cp tools/exp/lib_$v.so paper_2507_17245_b200/libdistr_attn.so; fi
  timeout -s KILL 600 python bench.py --no-e2e --no-cpu --no-parity --steps 10 > $O/bench_${v}_$rep.log 2>&1
  [ $rep = 1 ] && timeout -s KILL 60 python tools/trace.py distr > $O/trace_$v.log 2>&1
 done
done
cp /tmp/lib_default.so paper_2507_17245_b200/libdistr_attn.so
