#!/bin/bash
# A/B: sibling lockstep (phase 2) and L2 cache hints vs the default engine.
TAG=${1:-ab2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
SDMRG_LIB=paper_2305_05581_b200/lib/exp/lib_lock2.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $OUT/pytest_lock2.log 2>&1; echo "rc=$?" >> $OUT/pytest_lock2.log
V="default lock2 lock6 l2hint"
R="l2hint lock6 lock2 default"
for order in "$V" "$R"; do
  for v in $order; do
    for cfg in "50 4096" "30 2048"; do
      if [ $v = default ]; then L=""; else L=paper_2305_05581_b200/lib/exp/lib_$v.so; fi
      echo "[$v] $cfg: $(SDMRG_LIB=$L timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)" | cut -c1-260 >> $OUT/ab.log
    done
  done
done
ls -la $OUT
