# post-bundle check after a kernel change: GPU tests, smoke, the main bench lines, launch list
TAG=${1:-f8}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PYTHONDONTWRITEBYTECODE=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
for wl in hyperspectral weather tiny hyperspectral_linear; do
  timeout 600 python bench.py --workload $wl > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err
done
timeout 900 python bench.py --workload train > $OUT/bench_train.json 2> $OUT/bench_train.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"l0_|gemm_kernel|combine|child_softmax|unfold|vit_" -c 200 --csv --log-file $OUT/launches_h1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
tail -2 $OUT/pytest_gpu.log; tail -3 $OUT/smoke.log
for f in $OUT/bench_*.json; do python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],4), r.get('kernel'), r.get('frac'), (d.get('clocks') or {}).get('sm_mhz'))" $f; done
