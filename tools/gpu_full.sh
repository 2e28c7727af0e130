#!/bin/bash
# Full pass: GPU tests, smoke, bench (default), EMU A/B, sweep, timelines.
O=gpurun_out/${TAG:-full}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout -s KILL 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
for e in 3 4; do DA_EMU=$e timeout -s KILL 300 python bench.py --no-e2e --no-cpu --no-parity > $O/bench_emu$e.log 2>&1; done
timeout -s KILL 600 python tools/sweep.py > $O/sweep.json 2> $O/sweep.err
timeout -s KILL 60 python tools/trace.py distr > $O/trace_distr.log 2>&1
timeout -s KILL 60 python tools/trace.py exact > $O/trace_exact.log 2>&1
