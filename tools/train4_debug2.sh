#!/bin/bash
# Second pass: default steps/warmup, direct ranks (faulthandler on hang), then torchrun
O=gpurun_out/d4b; mkdir -p $O
for r in 0 1 2 3; do
  MASTER_ADDR=127.0.0.1 MASTER_PORT=29656 WORLD_SIZE=4 RANK=$r LOCAL_RANK=$r \
    timeout -s ABRT 240 python -X faulthandler bench.py --gpus 4 --workload train \
    > $O/direct_r$r.out 2> $O/direct_r$r.err &
done
wait
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29657 bench.py --gpus 4 --workload train > $O/torchrun.json 2> $O/torchrun.err
echo "rc=$?" >> $O/torchrun.err
echo done > $O/DONE
