#!/bin/bash
# prep-kernel hashing (DA_PREHASH=1) vs in-CTA hashing: quick parity both ways, hash/export parity
# tests, then per-config call times both ways.
O=gpurun_out/ph2; mkdir -p $O
for ph in 1 0; do DA_PREHASH=$ph timeout -s KILL 180 python tools/quick.py > $O/quick$ph.log 2>&1; echo "rc=$?" >> $O/quick$ph.log; done
DA_PREHASH=1 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fwd_exports.py -x -q -p no:cacheprovider > $O/pytest1.log 2>&1; echo "rc=$?" >> $O/pytest1.log
for ph in 0 1; do DA_PREHASH=$ph timeout -s KILL 600 python tools/sweep.py --no-error > $O/sweep_$ph.json 2> $O/sweep_$ph.err; done
