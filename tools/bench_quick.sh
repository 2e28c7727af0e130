O=gpurun_out; mkdir -p $O
timeout -s KILL 120 python bench.py --steps 5 --no-e2e --no-cpu --no-parity > $O/bench_q.log 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 120 -k "hash or C2 or C3 or ragged" > $O/pytest_sub.log 2>&1
