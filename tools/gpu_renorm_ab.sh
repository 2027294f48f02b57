#!/bin/bash
TAG=${1:-renormab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for order in "default noswz" "noswz default"; do
  for v in $order; do
    if [ $v = default ]; then L=""; else L=paper_2305_05581_b200/lib/exp/lib_$v.so; fi
    SDMRG_LIB=$L timeout 1200 python tools/sweep_run.py 24 1024 1 --model-seed 1 --scale 0.1 --core 0.0 > $OUT/sweep_$v.log 2>&1
    echo "[$v] $(tail -1 $OUT/sweep_$v.log | cut -c1-600)" >> $OUT/ab.log
  done
done
