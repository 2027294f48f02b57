#!/bin/bash
TAG=${1:-ab3}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
L2=paper_2305_05581_b200/lib/exp/lib_lock2.so
for r in 1 2; do
  for v in default nolock lock2 nolock default; do
    for cfg in "50 4096" "30 2048" "76 4096 113"; do
      case $v in
        default) out=$(timeout 600 python tools/quick.py $cfg 2>&1 | tail -1);;
        nolock) out=$(SDMRG_NO_LOCK=1 SDMRG_LIB=$L2 timeout 600 python tools/quick.py $cfg 2>&1 | tail -1);;
        lock2) out=$(SDMRG_LIB=$L2 timeout 600 python tools/quick.py $cfg 2>&1 | tail -1);;
      esac
      echo "[$v] $cfg: $out" | sed 's/"lib": "[^"]*", //' | cut -c1-220 >> $OUT/ab.log
    done
  done
done
timeout 900 python tools/quick.py 76 8192 113 > $OUT/quick_L76_D8192.log 2>&1
ls -la $OUT
