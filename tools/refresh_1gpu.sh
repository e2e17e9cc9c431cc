#!/bin/bash
# One-GPU measurement bundle (run via gpurun from the repo root): GPU tests, bench lines of
# every workload, ncu launch list and full captures of the hot kernels -> gpurun_out/r/
set -u
O=gpurun_out/r
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_h1.json 2> $O/bench_h1.err
for w in weather tiny train; do
  timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for w in sweep_c64_d1024 sweep_c128_d1024 sweep_c256_d1024 sweep_c512_d1024 sweep_c1024_d1024 \
         sweep_c64_d4096 sweep_c128_d4096 sweep_c256_d4096 sweep_c512_d4096 sweep_c1024_d4096; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline --steps 10 > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > $O/ncu_launch.log 2>&1
for k in l0_node_kernel gemm_kernel l0_logits_kernel combine_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -s 4 \
      -o $O/full_$k python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
      > $O/ncu_full_$k.log 2>&1
done
echo done > $O/DONE
