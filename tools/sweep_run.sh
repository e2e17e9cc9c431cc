#!/bin/bash
# the SURVEY 8(d) scaling sweep on one B200: C 64..1024 x D 1024 / 4096
OUT=gpurun_out/${1:-sw}; mkdir -p $OUT
for c in 64 128 256 512 1024; do for d in 1024 4096; do
  timeout 300 python bench.py --workload sweep_c${c}_d${d} --no-cpu-baseline --steps 10 > $OUT/sweep_c${c}_d${d}.json 2> $OUT/sweep_c${c}_d${d}.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d.get('roofline') or {}; print(sys.argv[1].split('/')[-1], round(d['value']), round(d['ms_per_step'],3), r.get('kernel'), r.get('frac') and round(r['frac'],3))" $OUT/sweep_c${c}_d${d}.json 2>/dev/null || (echo "sweep_c${c}_d${d} FAILED"; tail -3 $OUT/sweep_c${c}_d${d}.err)
done; done
