#!/bin/bash
OUT=gpurun_out/${1:-p3}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o $OUT/fcqk python bench.py --workload hyperspectral_fullcross --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu1.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:fullcross_weights -c 1 -o $OUT/fcw python bench.py --workload hyperspectral_fullcross --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu2.log 2>&1
