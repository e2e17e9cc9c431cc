# K_p0 copy issue: one lane per channel vs one thread (DCHAG_P0_ISSUE=1), H1 step, twice each
for i in 1 2; do for v in 0 1; do
DCHAG_P0_ISSUE=$v python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); ks={k['site']:k['ms'] for k in d['kernels']}
print('one warp' if '$v' == '1' else 'all warps', round(d['value']), round(d['ms_per_step'], 4), 'l0_logits', round(ks.get('l0_logits'), 4), 'l0_node', round(ks.get('l0_node'), 4))"
done; done
DCHAG_P0_ISSUE=1 python tools/p0_trace.py | tail -2; python tools/p0_trace.py | tail -2
