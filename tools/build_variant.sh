#!/bin/bash
# build an A/B variant of libdchag.so with extra nvcc flags into $1 (timing probes only)
# usage: bash tools/build_variant.sh paper_2506_21411_b200/libdchag_x.so -DDCHAG_MBAR_HINT=100000
OUT=$1; shift
D=$(mktemp -d)
for s in capi gemm l0 comb train; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       -diag-suppress 177 "$@" -c -o $D/$s.o paper_2506_21411_b200/csrc/$s.cu &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xlinker --no-undefined \
     -o $OUT $D/*.o && echo built $OUT
rm -rf $D
