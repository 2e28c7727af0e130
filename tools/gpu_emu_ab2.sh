#!/bin/bash
# DistrAttention EMU (FMA-pipe exp2 share) on the final kernel, alternating C5 benches.
O=gpurun_out/emu_ab2; mkdir -p $O
for rep in 1 2; do
  for e in 2 3 4; do
    DA_EMU=$e timeout -s KILL 600 python bench.py --no-e2e --no-cpu --no-parity --steps 10 > $O/bench_e${e}_$rep.log 2>&1
  done
done
