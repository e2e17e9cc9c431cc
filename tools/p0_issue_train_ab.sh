for i in 1 2; do for v in 0 1; do
DCHAG_P0_ISSUE=$v python bench.py --workload train --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); ks={k['site']:k['ms'] for k in d['kernels']}
print('$v', round(d['ms_per_step'], 3), 'l0_logits', round(ks.get('fwd:l0_logits'), 4))"
done; done
