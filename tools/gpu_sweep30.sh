#!/bin/bash
TAG=${1:-sweep30}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 3000 python tools/sweep_run.py 30 2048 1 --model-seed 1 --scale 0.1 --core 0.0 \
    --out $OUT/sweep_L30_D2048.jsonl > $OUT/sweep_L30_D2048.log 2>&1
ls -la $OUT
