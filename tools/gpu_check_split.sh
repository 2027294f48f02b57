#!/bin/bash
TAG=${1:-split}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -q -k "L76" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for r in 1 2; do
  for cfg in "76 4096 113" "50 4096" "30 1024"; do
    echo "[new] $cfg: $(timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)" | sed 's/"lib": "[^"]*", //' | cut -c1-200 >> $OUT/ab.log
  done
done
