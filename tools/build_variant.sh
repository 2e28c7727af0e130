#!/bin/bash
# Build an experimental variant of the library with extra nvcc flags into tools/exp/lib_<name>.so
# (same sources; used for A/B timing on the GPU box). Usage: tools/build_variant.sh name -DFLAG ...
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
O=$R/tools/exp/build_$name; mkdir -p $O
for f in api prep prep_global bwd bwd_fused attn; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I$R/include "$@" -c $R/paper_2507_17245_b200/csrc/$f.cu -o $O/$f.o -Xptxas -v 2> $O/$f.log &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/exp/lib_$name.so $O/api.o $O/prep.o $O/prep_global.o $O/bwd.o $O/bwd_fused.o $O/attn.o
echo $R/tools/exp/lib_$name.so
