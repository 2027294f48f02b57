#!/bin/bash
# Closed-loop device sweeps on one B200: the GPU sweep-parity tests and
# timed runs (records + sec/sweep) into gpurun_out/TAG.
TAG=${1:-sweep}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_closed_sweep.py -q -x > $OUT/pytest_sweep.log 2>&1; echo "rc=$?" >> $OUT/pytest_sweep.log
timeout 1200 python tools/sweep_run.py 16 256 4 --ref tests/golden/sweep_record_L16_D256.jsonl \
    --out $OUT/sweep_L16_D256.jsonl > $OUT/sweep_L16_D256.log 2>&1
shift
for cfg in "$@"; do
  set -- $cfg
  timeout 2400 python tools/sweep_run.py $1 $2 $3 --model-seed 1 --scale 0.1 --core 0.0 \
      --out $OUT/sweep_L$1_D$2.jsonl > $OUT/sweep_L$1_D$2.log 2>&1
done
ls -la $OUT
