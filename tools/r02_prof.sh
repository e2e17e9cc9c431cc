#!/bin/bash
# ncu captures of the training step's level-0 kernels and the full_cross path (one B200)
OUT=gpurun_out/${1:-p1}; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
python tools/rowdot_micro.py > $OUT/rowdot_micro.txt 2>&1
python tools/te_micro.py > $OUT/te_micro.txt 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o $OUT/rowdot python tools/rowdot_micro.py > $OUT/ncu_rowdot.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:l0_tgrad -s 3 -c 1 -o $OUT/te python tools/te_micro.py > $OUT/ncu_te.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:softmax_bwd -s 3 -c 1 -o $OUT/smbwd python bench.py --workload train --steps 1 --warmup 1 --no-graph --no-cpu-baseline > $OUT/ncu_smbwd.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:fullcross_weights -c 1 -o $OUT/fcw python bench.py --workload hyperspectral_fullcross --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_fcw.log 2>&1
cat $OUT/rowdot_micro.txt $OUT/te_micro.txt
