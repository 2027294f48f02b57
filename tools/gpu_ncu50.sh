#!/bin/bash
# ncu --set full of one phase-1 and one phase-2 launch (chunk 0 of the second apply) at L=50 D=4096
OUT=gpurun_out/${1:-n50b}; mkdir -p $OUT
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:seg_gemm_kernel -s 8 -c 2 \
    -o $OUT/prof python tools/prof_apply.py 50 4096 2 > $OUT/ncu.log 2>&1
tail -n 3 $OUT/ncu.log
