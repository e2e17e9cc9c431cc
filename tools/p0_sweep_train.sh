#!/bin/bash
# K_p0 (dchag_l0_logits) launch-shape sweep on the TR training step (DCHAG_P0_* overrides)
run() {
  env "$@" timeout 300 python bench.py --workload train --no-cpu-baseline --steps 5 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ks={k['site']:k['ms'] for k in d['kernels']}
print('$*', 'step', round(d['ms_per_step'],3), 'fwd', round(ks.get('fwd:l0_logits',0),3), 'bwd', round(ks.get('bwd:l0_logits',0),3))" 2>/dev/null || echo "$* failed"
}
run X=0
for rb in 16 32 64; do for nb in 1 2; do for ps in 1 2 3; do
  run DCHAG_P0_RB=$rb DCHAG_P0_NBUF=$nb DCHAG_P0_PERSM=$ps
done; done; done
