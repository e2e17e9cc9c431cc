#!/bin/bash
# lean-epilogue check: GPU tests + the H1 / full_cross / linear / train bench lines, with and
# without the lean epilogue (DCHAG_GEMM_LEAN=0)
TAG=${1:-lean}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for wl in hyperspectral hyperspectral_fullcross hyperspectral_linear train; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline > $OUT/$wl.json 2> $OUT/$wl.err
  DCHAG_GEMM_LEAN=0 timeout 600 python bench.py --workload $wl --no-cpu-baseline > $OUT/${wl}_nolean.json 2> $OUT/${wl}_nolean.err
  python - $OUT/$wl.json $OUT/${wl}_nolean.json <<'PY'
import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], d.get("roofline", {}).get("frac"))
    except Exception as e:
        print(f, "ERR", e)
PY
done
