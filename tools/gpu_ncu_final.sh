#!/bin/bash
# ncu of the final phase-2 kernels (64-tile and big-tile instances) at the
# bench workload, and the big-tile split granule A/B.
TAG=${1:-ncufinal}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"sdmrg::seg_gemm_kernel<.bool.0, .bool.0" -s 0 -c 1 \
    -o $OUT/prof_p2small python tools/prof_apply.py 50 4096 1 > $OUT/ncu_p2small.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:sdmrg_big -s 0 -c 1 -o $OUT/prof_p2big python tools/prof_apply.py 50 4096 1 > $OUT/ncu_p2big.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"sdmrg::seg_gemm_kernel<.bool.0, .bool.1" -s 0 -c 1 \
    -o $OUT/prof_p1 python tools/prof_apply.py 50 4096 1 > $OUT/ncu_p1.log 2>&1
for r in 1 2; do
  for v in 96 24 8; do
    for cfg in "50 4096" "76 8192 113"; do
      echo "[bsplit=$v] $cfg: $(SDMRG_BIG_SPLIT=$v timeout 900 python tools/quick.py $cfg 2>&1 | tail -1)" | sed 's/"lib": "[^"]*", //' | cut -c1-200 >> $OUT/ab.log
    done
  done
done
ls -la $OUT
