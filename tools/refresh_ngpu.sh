#!/bin/bash
# N-GPU measurement bundle (via gpurun --gpus N): NCCL parity + ledger, forward and training
# bench lines -> gpurun_out/n$N/
set -u
N=$1
O=gpurun_out/n$N
mkdir -p $O
run() { timeout "$1" python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
          --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
run 600 29611 tools/dist_parity.py > $O/dist_parity.log 2>&1; echo "rc=$?" >> $O/dist_parity.log
run 600 29612 bench.py --gpus $N > $O/bench_fwd.json 2> $O/bench_fwd.err
run 600 29613 bench.py --gpus $N --workload train > $O/bench_train.json 2> $O/bench_train.err
run 600 29614 bench.py --gpus $N --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
cp gpurun_out/ledger_tp*.csv $O/ 2>/dev/null
echo done > $O/DONE
