#!/bin/bash
# Iteration pass: quick check (fail fast), parity subset, bench (no e2e / cpu), CTA-0 timelines,
# per-config sweep. TAG names the output dir; SKIP_TESTS=1 skips pytest.
O=gpurun_out/${TAG:-iter}; mkdir -p $O
timeout -s KILL 180 python tools/quick.py > $O/quick.log 2>&1; rc=$?; echo "quick rc=$rc" >> $O/quick.log
if [ $rc -ne 0 ]; then exit 0; fi
timeout -s KILL 60 python tools/trace.py distr > $O/trace_distr.log 2>&1
timeout -s KILL 60 python tools/trace.py exact > $O/trace_exact.log 2>&1
timeout -s KILL 600 python bench.py --no-e2e --no-cpu > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout -s KILL 600 python tools/sweep.py > $O/sweep.json 2> $O/sweep.err
if [ -z "$SKIP_TESTS" ]; then
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fwd_exports.py -x -q -p no:cacheprovider ${PYTEST_ARGS} > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
fi
