# ncu --set full of one TR-shaped TE launch (tools/te_micro.py)
mkdir -p gpurun_out/ep
python tools/te_micro.py && \
ncu --set full --import-source on --clock-control none -k regex:l0_tgrad --launch-skip 2 -c 1 \
    -o gpurun_out/ep/te -f python tools/te_micro.py > gpurun_out/ep/ncu_te.log 2>&1
tail -1 gpurun_out/ep/ncu_te.log
