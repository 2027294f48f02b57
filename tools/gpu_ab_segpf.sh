#!/bin/bash
TAG=${1:-abseg}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for order in "default segpf4" "segpf4 default"; do
  for v in $order; do
    for cfg in "76 4096 113" "50 4096" "30 1024"; do
      if [ $v = default ]; then L=""; else L=paper_2305_05581_b200/lib/exp/lib_$v.so; fi
      echo "[$v] $cfg: $(SDMRG_LIB=$L timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)" | sed 's/"lib": "[^"]*", //' | cut -c1-200 >> $OUT/ab.log
    done
  done
done
