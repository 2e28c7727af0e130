#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full captures (forward attention, K^T
# prep, fused backward), per-config sweep, Pareto sweep, backward timing. Logs under gpurun_out/.
set -x
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
if [[ "$1" != "nobench-tests" ]]; then
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout -s KILL 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prep_kernel|attn_kernel|convert_kernel" -c 60 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_launches.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 3 -c 1 -o $O/prof_attn -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_full_attn.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:prep_kernel -s 3 -c 1 -o $O/prof_prep -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_full_prep.log 2>&1
# summaries on the box (the .ncu-rep files with source are too large to ship back)
for k in attn prep; do
  python tools/ncu_summary.py $O/prof_$k.ncu-rep $O/ncu_$k > $O/ncu_summary_$k.log 2>&1
  ncu -i $O/prof_$k.ncu-rep --page source --csv --print-source sass > $O/ncu_${k}_sass.csv 2>&1
  python tools/sass_stalls.py $O/ncu_${k}_sass.csv > $O/ncu_${k}_stalls.txt 2>&1
  rm -f $O/prof_$k.ncu-rep $O/ncu_${k}_sass.csv
done
timeout -s KILL 60 python tools/trace.py distr > $O/trace_distr.log 2>&1
timeout -s KILL 60 python tools/trace.py exact > $O/trace_exact.log 2>&1
timeout -s KILL 600 python tools/sweep.py > $O/sweep.json 2> $O/sweep.err
timeout -s KILL 600 python tools/sweep.py --only "C4 N=16384,C4 N=32768,C4 N=65536,C5" --block-l 256 > $O/sweep_l256.json 2> $O/sweep_l256.err
timeout -s KILL 1500 python tools/pareto.py > $O/pareto.json 2> $O/pareto.err
timeout -s KILL 600 python tools/bench_bwd.py > $O/bwd.json 2> $O/bwd.err
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kv_kernel|bwd_q_kernel" -c 2 -o $O/prof_bwd -f python tools/bench_bwd.py > $O/ncu_full_bwd.log 2>&1
python tools/ncu_summary.py $O/prof_bwd.ncu-rep $O/ncu_bwd > $O/ncu_summary_bwd.log 2>&1; rm -f $O/prof_bwd.ncu-rep
ls -la $O
