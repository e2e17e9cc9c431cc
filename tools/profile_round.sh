#!/bin/bash
# Round profile bundle (run on the GPU box via gpurun, from the repo root):
#   1. bench.py default line                      -> gpurun_out/bench.json
#   2. ncu launch list of a short bench run       -> gpurun_out/launches.csv
#   3. ncu --set full of one launch per hot kernel -> gpurun_out/full_<kernel>.ncu-rep
set -u
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launch.log 2>&1
for k in l0_node_kernel gemm_kernel l0_logits_kernel combine_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -s 4 \
      -o gpurun_out/full_$k python tools/profile_step.py --batch 32 --iters 3 \
      > gpurun_out/ncu_full_$k.log 2>&1
done
echo done
