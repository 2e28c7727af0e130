#!/bin/bash
# Multi-rank bench path on a 1-GPU box: 2 and 3 ranks share cuda:0 (gloo), batch and flattened-head
# shards, and the Q-pair shard mode; each prints rank 0's JSON line.
O=gpurun_out/${TAG:-mr}; mkdir -p $O
for n in 2 3; do
  BENCH_SHARE_GPU=1 timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 2 --warmup 3 --no-e2e --no-cpu > $O/bench_share$n.log 2>&1; echo "rc=$?" >> $O/bench_share$n.log
done
BENCH_SHARE_GPU=1 timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 2 --warmup 3 --no-e2e --no-cpu --shard q > $O/bench_share2_q.log 2>&1; echo "rc=$?" >> $O/bench_share2_q.log
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > $O/bench_ref2.log 2>&1; echo "rc=$?" >> $O/bench_ref2.log
