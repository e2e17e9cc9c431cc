#!/bin/bash
OUT=gpurun_out/g4b; mkdir -p $OUT
for mode in group default; do
  PROBE_MODE=$mode timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) tools/graph4_probe2.py \
    > $OUT/$mode.log 2>&1
  echo "$mode exit $?"; grep -o "\[$mode\] rank [0-9]: [a-z_ +]*OK" $OUT/$mode.log | sort | uniq -c
done
