#!/bin/bash
# full_cross check: its GPU tests + the H1 full_cross bench line (kernel table)
TAG=${1:-fc}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "full_cross or fullcross or fc" > $OUT/pytest_fc.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_fc.log
tail -2 $OUT/pytest_fc.log
timeout 600 python bench.py --workload hyperspectral_fullcross --no-cpu-baseline > $OUT/fc.json 2> $OUT/fc.err
python - $OUT/fc.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("fc", round(d["value"], 1), "img/s", round(d["ms_per_step"], 3), "ms", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3))
for k in sorted(d["kernels"], key=lambda k: -k["ms"])[:10]:
    print(f"  {k['site']:24s} {k['kernel']:26s} {k['ms']:7.3f} ms x{k['launches']:.0f}")
PY
