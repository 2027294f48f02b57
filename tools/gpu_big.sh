#!/bin/bash
TAG=${1:-big}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
SDMRG_BIG=1 timeout 900 python -m pytest tests/test_gpu_bench_parity.py -q -x -k "L30_D2048 or L50" > $OUT/pytest_big.log 2>&1; echo "rc=$?" >> $OUT/pytest_big.log
for r in 1 2; do
  for v in 0 1; do
    for cfg in "50 4096" "30 2048"; do
      echo "[big=$v] $cfg: $(SDMRG_BIG=$v timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)" | sed 's/"lib": "[^"]*", //' | cut -c1-220 >> $OUT/ab.log
    done
  done
done
SDMRG_BIG=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:sdmrg_big -s 1 -c 1 \
    -o $OUT/prof_big python tools/prof_apply.py 50 4096 2 > $OUT/ncu_big.log 2>&1
for v in 1 0; do
  echo "[big=$v] 76 8192: $(SDMRG_BIG=$v timeout 900 python tools/quick.py 76 8192 113 2>&1 | tail -1)" | cut -c1-220 >> $OUT/ab.log
done
ls -la $OUT
for ws in 11250000000 0; do
  echo "[ws=$ws] 50 4096: $(SDMRG_WS=$ws timeout 600 python tools/quick.py 50 4096 2>&1 | tail -1)" | cut -c1-220 >> $OUT/ab.log
done
