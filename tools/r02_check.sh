#!/bin/bash
# round-2 GPU check bundle: GPU tests, smoke, the default bench line and the training line.
# usage (from the repo root, on a GPU box): bash tools/r02_check.sh TAG
TAG=${1:-v1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_h1.json 2> $OUT/bench_h1.err
timeout 600 python bench.py --workload train --no-cpu-baseline > $OUT/bench_train.json 2> $OUT/bench_train.err
tail -3 $OUT/pytest_gpu.log
cat $OUT/smoke.log | tail -3
head -c 600 $OUT/bench_h1.json; echo
head -c 600 $OUT/bench_train.json; echo
