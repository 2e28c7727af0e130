O=gpurun_out; mkdir -p $O
timeout -s KILL 60 compute-sanitizer --tool memcheck python tools/diag1.py 300 128 128 1 0 0 > $O/memcheck.log 2>&1
for cfg in "300 128 128 1 0 0" "300 128 128 4 0 0" "300 128 64 2 0 0" "300 64 128 2 0 0" "300 64 64 2 0 0" "300 64 64 1 0 0" "1000 128 128 2 1 0" "1000 128 128 2 1 1" "1000 64 128 1 0 0"; do timeout -s KILL 30 python tools/diag1.py $cfg >> $O/cfgs.log 2>&1 || echo "FAIL $cfg rc=$?" >> $O/cfgs.log; done
