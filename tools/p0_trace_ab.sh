# H1 step, three runs, per-site times of the level-0 kernels
for i in 1 2 3; do
python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); ks={k['site']:k['ms'] for k in d['kernels']}
print(round(d['value']), round(d['ms_per_step'], 4), 'l0_logits', round(ks.get('l0_logits'), 4), 'l0_node', round(ks.get('l0_node'), 4), 'comb', round(ks.get('gemm_combine_l0'), 4))"
done
