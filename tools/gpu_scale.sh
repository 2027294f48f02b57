#!/bin/bash
# Larger closed-loop sweeps and the D=8192 north-star scale point.
TAG=${1:-scale}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python tools/scale_point.py 76 8192 113 > $OUT/scale_L76_D8192.log 2>&1
timeout 2400 python tools/sweep_run.py 30 2048 1 --model-seed 1 --scale 0.1 --core 0.0 \
    --out $OUT/sweep_L30_D2048.jsonl > $OUT/sweep_L30_D2048.log 2>&1
timeout 1200 python tools/sweep_run.py 16 256 2 --ref tests/golden/sweep_record_L16_D256.jsonl \
    --out $OUT/sweep_L16_D256.jsonl > $OUT/sweep_L16_D256.log 2>&1
ls -la $OUT
