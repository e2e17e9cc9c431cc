#!/bin/bash
# Second pass: default steps/warmup, direct ranks (faulthandler on hang), then torchrun
O=gpurun_out/d4c; mkdir -p $O
for r in 0 1 2 3; do
  OMP_NUM_THREADS=1 MASTER_ADDR=127.0.0.1 MASTER_PORT=29656 WORLD_SIZE=4 RANK=$r LOCAL_RANK=$r \
    timeout -s ABRT 200 python -X faulthandler bench.py --gpus 4 --workload train \
    > $O/direct_r$r.out 2> $O/direct_r$r.err &
done
wait
echo done > $O/DONE
