# ncu --set full of the K = 64 q | k GEMM (tools/ncu_gemm_one.py); run under gpurun
mkdir -p gpurun_out/ep
python tools/ncu_gemm_one.py && \
ncu --set full --import-source on --clock-control none -k regex:gemm_kernel --launch-skip 3 -c 1 \
    -o gpurun_out/ep/gemm_k64 -f python tools/ncu_gemm_one.py > gpurun_out/ep/ncu.log 2>&1
tail -3 gpurun_out/ep/ncu.log
