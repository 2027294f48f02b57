#!/bin/bash
TAG=${1:-sweepsf}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 1500 python tools/sweep_run.py 16 256 2 --ref tests/golden/sweep_record_L16_D256.jsonl \
    --out $OUT/sweep_L16_D256.jsonl > $OUT/sweep_L16_D256.log 2>&1
timeout 2400 python tools/sweep_run.py 30 1024 1 --model-seed 1 --scale 0.1 --core 0.0 \
    --out $OUT/sweep_L30_D1024.jsonl > $OUT/sweep_L30_D1024.log 2>&1
ls -la $OUT
