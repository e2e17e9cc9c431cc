# ncu --set full (source counters) of one full_cross level-0 weights launch (H1 shape)
mkdir -p gpurun_out/ep
python bench.py --workload hyperspectral_fullcross --no-cpu-baseline --steps 2 --warmup 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:fullcross_weights --launch-skip 2 -c 1 \
    -o gpurun_out/ep/fcw -f python bench.py --workload hyperspectral_fullcross --no-cpu-baseline \
    --steps 1 --warmup 1 > gpurun_out/ep/ncu_fcw.log 2>&1
tail -2 gpurun_out/ep/ncu_fcw.log
