#!/bin/bash
# multi-GPU bundle: NCCL parity, forward and training bench lines at N GPUs (one box)
N=${1:-4}
TAG=${2:-m1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
run() { timeout ${1} python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) ${@:2}; }
run 600 tools/dist_parity.py > $OUT/dist_parity_$N.log 2>&1; echo "parity exit $?" >> $OUT/dist_parity_$N.log
run 600 bench.py --gpus $N > $OUT/bench_h$N.json 2> $OUT/bench_h$N.err
run 900 bench.py --gpus $N --workload train --steps 10 > $OUT/bench_train$N.json 2> $OUT/bench_train$N.err; echo "train exit $?" >> $OUT/bench_train$N.err
tail -2 $OUT/dist_parity_$N.log
head -c 300 $OUT/bench_h$N.json; echo
head -c 300 $OUT/bench_train$N.json; echo
tail -3 $OUT/bench_train$N.err
