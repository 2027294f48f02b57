#!/bin/bash
# L=76 (CAS(113,76)) per-phase timing, rotation A/B and ncu captures of the
# two engine phases: tools/gpu_l76.sh TAG
TAG=${1:-l76}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
NOTEST=1 CFGS="76 4096 113;50 4096" timeout 1500 bash tools/ab_lib.sh $TAG default norot > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm_kernel -s 2 -c 1 \
    -o $OUT/prof_p1 python tools/prof_apply.py 76 4096 2 113 > $OUT/ncu_p1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm_kernel -s 3 -c 1 \
    -o $OUT/prof_p2 python tools/prof_apply.py 76 4096 2 113 > $OUT/ncu_p2.log 2>&1
ls -la $OUT
