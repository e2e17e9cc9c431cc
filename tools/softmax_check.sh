# child softmax in registers: GPU tests touching it + H1 step per-site times
timeout 500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_shapes.py tests/test_gpu_train.py tests/test_capi.py -x -q -m gpu 2>&1 | tail -1
for i in 1 2 3; do
python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); ks={k['site']:k['ms'] for k in d['kernels']}
print(round(d['value']), round(d['ms_per_step'], 4), 'softmax_l1', round(ks.get('child_softmax_l1'), 4), 'softmax_l2', round(ks.get('child_softmax_l2'), 4))"
done
