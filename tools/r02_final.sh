#!/bin/bash
# round-2 GPU evidence bundle (one B200): GPU tests, smoke, every bench workload, ncu launch
# list + full captures of the dominant kernels, compute-sanitizer logs, cost-model validation.
TAG=${1:-f1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONDONTWRITEBYTECODE=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
for wl in hyperspectral weather tiny hyperspectral_linear hyperspectral_fullcross hyperspectral_fp32; do
  timeout 600 python bench.py --workload $wl > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
timeout 900 python bench.py --workload train > $OUT/bench_train.json 2> $OUT/bench_train.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for n in 2 4 8; do timeout 600 python bench.py --arch-tp $n --no-cpu-baseline > $OUT/bench_arch$n.json 2> $OUT/bench_arch$n.err; done
timeout 900 python tools/costmodel_validate.py > $OUT/costmodel_validate.json 2> $OUT/costmodel_validate.err
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -k regex:"l0_|gemm_kernel|combine|child_softmax|unfold|vit_" -c 200 --csv --log-file $OUT/launches_h1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:l0_node_kernel -c 1 -o $OUT/l0_node python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_l0.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 -o $OUT/gemm python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_gemm.log 2>&1
timeout 900 $NCU --set full --clock-control none -k regex:gemm_kernel -c 3 -o $OUT/train_gemm python bench.py --workload train --steps 1 --warmup 1 --no-graph --no-cpu-baseline > $OUT/ncu_train.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_t.py > $OUT/sanitize_$tool.log 2>&1; echo "exit $?" >> $OUT/sanitize_$tool.log
done
tail -3 $OUT/pytest_gpu.log; tail -3 $OUT/smoke.log
for f in $OUT/bench_*.json; do echo $f; head -c 250 $f; echo; done
for tool in memcheck racecheck synccheck; do tail -3 $OUT/sanitize_$tool.log; done
