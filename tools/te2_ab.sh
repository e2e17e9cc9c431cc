# K_te one- vs two-channel CTAs on the TR training step (A/B by DCHAG_TE_CH)
mkdir -p gpurun_out/te2
timeout 120 python tools/te_micro.py 0 3
timeout 600 python -m pytest tests/test_gpu_train.py -x -q -m gpu 2>&1 | tail -2
for i in 1 2; do
  for ch in 2 1; do
    DCHAG_TE_CH=$ch timeout 600 python bench.py --workload train --no-cpu-baseline > gpurun_out/te2/train_ch$ch.$i.json 2> gpurun_out/te2/train_ch$ch.$i.err
    python -c "
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
ks={k['site']:k['ms'] for k in d.get('kernels',[])}
print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],3), 'te', ks.get('bwd:l0_tgrad_te'))" gpurun_out/te2/train_ch$ch.$i.json
  done
done
