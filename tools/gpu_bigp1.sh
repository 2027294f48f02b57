#!/bin/bash
TAG=${1:-bigp1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -q -x -k "L30_D2048 or L50" > $OUT/pytest_bench.log 2>&1; echo "rc=$?" >> $OUT/pytest_bench.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $OUT/pytest_parity.log 2>&1; echo "rc=$?" >> $OUT/pytest_parity.log
for r in 1 2; do
  for v in 1 0; do
    for cfg in "50 4096" "30 2048" "76 8192 113"; do
      echo "[bigp1=$v] $cfg: $(SDMRG_BIG_P1=$v timeout 900 python tools/quick.py $cfg 2>&1 | tail -1)" | sed 's/"lib": "[^"]*", //' | cut -c1-200 >> $OUT/ab.log
    done
  done
done
timeout 600 python tools/lanczos_prof.py 50 4096 > $OUT/lanczos_prof_L50.log 2>&1
timeout 600 python tools/lanczos_prof.py 30 2048 > $OUT/lanczos_prof_L30.log 2>&1
ls -la $OUT
