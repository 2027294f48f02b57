#!/bin/bash
TAG=${1:-fused4}
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
timeout 1500 python -m pytest tests/test_gpu_closed_sweep.py -q > $OUT/pytest_sweep.log 2>&1; echo "rc=$?" >> $OUT/pytest_sweep.log
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -q -k "L76 or L30_D1024" > $OUT/pytest_bench_parity.log 2>&1; echo "rc=$?" >> $OUT/pytest_bench_parity.log
ls -la $OUT
