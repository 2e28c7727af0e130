#!/bin/bash
# Round-2 evidence pass on one build: GPU tests, smoke, bench line, sweeps (block_l 128 with the
# planner's pick, block_l 256), backward timings, ncu launch list + full captures + traffic json,
# sanitizers, CTA timelines.
O=gpurun_out/${TAG:-r2}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout -s KILL 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout -s KILL 900 python tools/sweep.py --plan > $O/sweep.json 2> $O/sweep.err
timeout -s KILL 900 python tools/sweep.py --block-l 256 > $O/sweep_l256.json 2> $O/sweep_l256.err
timeout -s KILL 600 python tools/bench_bwd.py > $O/bwd.json 2> $O/bwd.err
timeout -s KILL 60 python tools/trace.py distr > $O/trace_distr.log 2>&1
timeout -s KILL 60 python tools/trace.py exact > $O/trace_exact.log 2>&1
TAG=${TAG:-r2} bash tools/gpu_prof2.sh > /dev/null 2>&1
