#!/bin/bash
# Full ncu capture of one phase-2 engine launch (and one combine launch).
OUT=gpurun_out/${1:-p2}
mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:seg_gemm_kernel -s 3 -c 1 \
    -o $OUT/prof_p2 python tools/prof_apply.py 30 2048 3 > $OUT/ncu_p2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:combine -s 1 -c 1 \
    -o $OUT/prof_comb python tools/prof_apply.py 30 2048 2 > $OUT/ncu_comb.log 2>&1
tail -3 $OUT/ncu_p2.log $OUT/ncu_comb.log
