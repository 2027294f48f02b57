#!/bin/bash
TAG=${1:-abp1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
SDMRG_BIG_P1=2 timeout 600 python -m pytest tests/test_gpu_bench_parity.py -q -x -k "L30_D2048" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for order in "1 2" "2 1"; do
  for v in $order; do
    for cfg in "30 2048" "30 4096" "50 4096"; do
      echo "[bigp1=$v] $cfg: $(SDMRG_BIG_P1=$v timeout 900 python tools/quick.py $cfg 2>&1 | tail -1)" | sed 's/"lib": "[^"]*", //' | cut -c1-200 >> $OUT/ab.log
    done
  done
done
