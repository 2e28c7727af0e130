#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout -s KILL 60 python tools/diag.py hash exact > $O/diag.log 2>&1 || { echo "diag exact failed/hung rc=$?" >> $O/diag.log; exit 1; }
timeout -s KILL 60 python tools/diag.py distr >> $O/diag.log 2>&1 || { echo "diag distr failed/hung rc=$?" >> $O/diag.log; exit 1; }
timeout -s KILL 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 120 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for e in 0 2 3 4; do DA_EMU=$e timeout -s KILL 120 python bench.py --steps 5 --no-e2e --no-cpu --no-parity > $O/bench_emu$e.log 2>&1; done
