#!/bin/bash
TAG=${1:-big2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q > $OUT/pytest_parity.log 2>&1; echo "rc=$?" >> $OUT/pytest_parity.log
timeout 900 python -m pytest tests/test_gpu_closed_sweep.py -q -k "davidson or L8" > $OUT/pytest_davidson.log 2>&1; echo "rc=$?" >> $OUT/pytest_davidson.log
SDMRG_BIG=2 timeout 900 python -m pytest tests/test_gpu_bench_parity.py -q -x -k "L30_D2048 or L50" > $OUT/pytest_big2.log 2>&1; echo "rc=$?" >> $OUT/pytest_big2.log
for r in 1 2; do
  for v in 1 2 0; do
    for cfg in "50 4096" "30 2048" "76 4096 113"; do
      echo "[big=$v] $cfg: $(SDMRG_BIG=$v timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)" | sed 's/"lib": "[^"]*", //' | cut -c1-200 >> $OUT/ab.log
    done
  done
done
for v in 2 1; do
  echo "[big=$v] 76 8192: $(SDMRG_BIG=$v timeout 900 python tools/quick.py 76 8192 113 2>&1 | tail -1)" | cut -c1-220 >> $OUT/ab.log
done
ls -la $OUT
