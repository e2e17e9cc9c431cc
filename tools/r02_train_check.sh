#!/bin/bash
# training-path check: GPU train / parity tests + the TR bench line (kernel table)
TAG=${1:-tc}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py --workload train --no-cpu-baseline > $OUT/train.json 2> $OUT/train.err
python - $OUT/train.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("train", round(d["value"], 1), "img/s", round(d["ms_per_step"], 3), "ms", d["roofline"])
for k in sorted(d["kernels"], key=lambda k: -k["ms"])[:16]:
    print(f"  {k['site']:22s} {k['kernel']:26s} {k['ms']:7.3f} ms x{k['launches']:.0f}")
PY
