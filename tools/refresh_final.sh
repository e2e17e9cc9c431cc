#!/bin/bash
# Short one-GPU refresh: headline / weather / train bench lines, smoke, GPU tests,
# launch list -> gpurun_out/f/
set -u
O=gpurun_out/f
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_h1.json 2> $O/bench_h1.err
timeout 600 python bench.py --workload weather > $O/bench_weather.json 2> $O/bench_weather.err
timeout 600 python bench.py --workload train > $O/bench_train.json 2> $O/bench_train.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"l0_node|gemm_kernel|l0_logits|combine_kernel|child_softmax" -c 200 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > $O/ncu_launch.log 2>&1
timeout 300 python tools/train_profile.py > $O/train_profile.txt 2>&1
echo done > $O/DONE
