#!/bin/bash
# two-GPU bundle: NCCL parity, H2 forward, TR at 2 ranks, and the tp=2 architecture on one GPU
OUT=gpurun_out/${1:-m2}; mkdir -p $OUT
run() { timeout ${1} python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) ${@:2}; }
run 600 tools/dist_parity.py > $OUT/dist_parity_2.log 2>&1; echo "parity exit $?" >> $OUT/dist_parity_2.log
run 600 bench.py --gpus 2 > $OUT/bench_h2.json 2> $OUT/bench_h2.err
run 600 bench.py --gpus 2 --impl reference --steps 3 --warmup 1 > $OUT/bench_ref2.json 2> $OUT/bench_ref2.err
run 900 bench.py --gpus 2 --workload train > $OUT/bench_train2.json 2> $OUT/bench_train2.err
timeout 600 python bench.py --arch-tp 2 --no-cpu-baseline > $OUT/bench_arch2.json 2> $OUT/bench_arch2.err
tail -1 $OUT/dist_parity_2.log; for f in $OUT/bench_*.json; do echo $f; head -c 200 $f; echo; done
