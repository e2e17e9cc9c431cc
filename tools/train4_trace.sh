#!/bin/bash
OUT=gpurun_out/t4; mkdir -p $OUT
DCHAG_BENCH_TRACE=1 timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --workload train --steps 5 \
  --warmup 3 > $OUT/train4.json 2> $OUT/train4.err
echo "exit $?"; grep "\[bench rank" $OUT/train4.err | tail -40; head -c 400 $OUT/train4.json
