#!/bin/bash
OUT=gpurun_out/t4b; mkdir -p $OUT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29612 bench.py --gpus 4 --workload train > $OUT/train4.json 2> $OUT/train4.err
echo "exit $?"; head -c 600 $OUT/train4.json; echo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29613 bench.py --gpus 2 --workload train > $OUT/train2.json 2> $OUT/train2.err
echo "exit $?"; head -c 600 $OUT/train2.json; echo
