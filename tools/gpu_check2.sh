#!/bin/bash
# Quick check + backward + sweep after a build change.
O=gpurun_out/${TAG:-c2}; mkdir -p $O
timeout -s KILL 180 python tools/quick.py > $O/quick.log 2>&1; echo "quick rc=$?" >> $O/quick.log
timeout -s KILL 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout -s KILL 600 python tools/bench_bwd.py > $O/bwd.json 2> $O/bwd.err
timeout -s KILL 900 python tools/sweep.py > $O/sweep.json 2> $O/sweep.err
DA_PDL=0 timeout -s KILL 900 python tools/sweep.py --only "C1,C2,C3,C4 N=4096,C4 N=8192" > $O/sweep_nopdl.json 2> $O/sweep_nopdl.err
