# ncu --set full of the TR row-dot GEMM (tools/ncu_rowdot_one.py); run under gpurun
mkdir -p gpurun_out/ep
python tools/ncu_rowdot_one.py && \
ncu --set full --import-source on --clock-control none -k regex:gemm_kernel --launch-skip 3 -c 1 \
    -o gpurun_out/ep/rowdot -f python tools/ncu_rowdot_one.py > gpurun_out/ep/ncu_rowdot.log 2>&1
tail -2 gpurun_out/ep/ncu_rowdot.log
