mkdir -p gpurun_out/p0
for rb in 16 32 64 128; do for nb in 1 2; do
  DCHAG_P0_RB=$rb DCHAG_P0_NBUF=$nb timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/p0/rb${rb}_nb${nb}.json 2> gpurun_out/p0/rb${rb}_nb${nb}.err
done; done
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/p0/default.json 2> gpurun_out/p0/default.err
