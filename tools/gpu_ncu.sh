#!/bin/bash
# Full ncu captures of one phase-1 and one phase-2 engine launch at bench scale.
OUT=gpurun_out/${1:-ncu}
L=${2:-30}; D=${3:-2048}
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm_kernel -s 2 -c 1 \
    -o $OUT/prof_p1 python tools/prof_apply.py $L $D 2 > $OUT/ncu_p1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm_kernel -s 3 -c 1 \
    -o $OUT/prof_p2 python tools/prof_apply.py $L $D 2 > $OUT/ncu_p2.log 2>&1
tail -n 2 $OUT/ncu_p1.log $OUT/ncu_p2.log
