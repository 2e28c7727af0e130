#!/bin/bash
# Short end-of-session pass: GPU tests, smoke, bench line, ncu launch list of the bench command,
# per-config sweep (+ the block_l = 256 subset), CTA-0 timelines.
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout -s KILL 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout -s KILL 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prep_kernel|attn_kernel|convert_kernel" -c 60 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_launches.log 2>&1
timeout -s KILL 600 python tools/sweep.py > $O/sweep.json 2> $O/sweep.err
timeout -s KILL 600 python tools/sweep.py --only "C2,C3,C4 N=16384,C4 N=32768,C4 N=65536,C5" --block-l 256 > $O/sweep_l256.json 2> $O/sweep_l256.err
timeout -s KILL 60 python tools/trace.py distr > $O/trace_distr.log 2>&1
timeout -s KILL 60 python tools/trace.py exact > $O/trace_exact.log 2>&1
ls -la $O
