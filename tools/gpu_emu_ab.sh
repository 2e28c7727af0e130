#!/bin/bash
# EMU settings of the in-tree build (env overrides DA_EMU / DA_EMU_EXACT), alternating, C5 bench
# (kernel-only) + C4-16k sweep row; then the full GPU test suite on the in-tree build.
O=gpurun_out/emu_ab; mkdir -p $O
for rep in 1 2; do
  for cfg in "2 0" "2 2" "3 0" "3 3"; do
    set -- $cfg
    DA_EMU=$1 DA_EMU_EXACT=$2 timeout -s KILL 600 python bench.py --no-e2e --no-cpu --no-parity --steps 10 > $O/bench_$1_$2_$rep.log 2>&1
  done
done
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
