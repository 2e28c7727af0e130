#!/bin/bash
# Backward A/B: default build vs the variants in tools/exp (copied over the in-tree library in the
# box's scratch copy), tools/bench_bwd.py each, plus the backward parity tests on the default build.
O=gpurun_out/bwd_ab; mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_gpu_backward.py -x -q -p no:cacheprovider > $O/pytest_bwd.log 2>&1; echo "rc=$?" >> $O/pytest_bwd.log
timeout -s KILL 300 python tools/bench_bwd.py > $O/bwd_default.json 2>&1
cp paper_2507_17245_b200/libdistr_attn.so /tmp/lib_default.so
for v in "$@"; do
  cp tools/exp/lib_$v.so paper_2507_17245_b200/libdistr_attn.so
  timeout -s KILL 300 python tools/bench_bwd.py > $O/bwd_$v.json 2>&1
done
cp /tmp/lib_default.so paper_2507_17245_b200/libdistr_attn.so
timeout -s KILL 300 python tools/bench_bwd.py > $O/bwd_default2.json 2>&1
