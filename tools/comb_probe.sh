for dbg in 0 8 2; do
  DCHAG_GEMM_DEBUG=$dbg timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ks={k['site']:k['ms'] for k in d['kernels']}
print('debug=$dbg', 'step', round(d['ms_per_step'],3), 'comb_l0', round(ks.get('gemm_combine_l0',0),3), 'comb_l1', round(ks.get('gemm_combine_l1',0),3), 'logits_l0', round(ks.get('gemm_logits_l0',0),3))"
done
