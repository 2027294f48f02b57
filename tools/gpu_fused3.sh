#!/bin/bash
# Fused kernel v2 (warps split sigma columns, 2 CTAs/SM) + engine swizzle A/B.
TAG=${1:-fused3}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $OUT/pytest_parity.log 2>&1; echo "rc=$?" >> $OUT/pytest_parity.log
for cfg in "76 4096 113" "50 4096" "30 1024"; do
  for f in 1 0; do
    echo "[fused=$f] $cfg: $(SDMRG_FUSED=$f timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)" >> $OUT/quick.log
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_heff -c 1 \
    -o $OUT/prof_fused python tools/prof_apply.py 76 4096 1 113 > $OUT/ncu_fused.log 2>&1
SDMRG_FUSED=0 SDMRG_LIB=paper_2305_05581_b200/lib/exp/lib_swz.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $OUT/pytest_parity_swz.log 2>&1; echo "rc=$?" >> $OUT/pytest_parity_swz.log
for r in 1 2; do
  for v in default swz; do
    for cfg in "30 2048" "50 4096"; do
      if [ $v = default ]; then L=""; else L=paper_2305_05581_b200/lib/exp/lib_swz.so; fi
      echo "[$v] $cfg: $(SDMRG_FUSED=0 SDMRG_LIB=$L timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)" >> $OUT/ab_swz.log
    done
  done
done
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -q -k "L76 or L30_D1024" > $OUT/pytest_bench_parity.log 2>&1; echo "rc=$?" >> $OUT/pytest_bench_parity.log
ls -la $OUT
