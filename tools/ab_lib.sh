#!/bin/bash
# A/B of two builds of the library (default vs $1) on the GEMM probes and the H1 / train lines
ALT=$1
OUT=gpurun_out/ab
mkdir -p $OUT
for lib in "" "$ALT"; do
  echo "== lib ${lib:-default}"
  DCHAG_LIB=$lib python tools/rowdot_probe.py 2>&1 | head -1
  DCHAG_LIB=$lib python tools/gemm_epi_probe.py 2>&1 | head -1
  for wl in hyperspectral train; do
    DCHAG_LIB=$lib timeout 600 python bench.py --workload $wl --no-cpu-baseline > $OUT/$wl$( [ -n "$lib" ] && echo _alt).json 2>/dev/null
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],1), round(d['ms_per_step'],3), d['roofline'].get('frac'))" $OUT/$wl$( [ -n "$lib" ] && echo _alt).json
  done
done
