#!/bin/bash
# configs[4] D sweep at L=30 and the CAS(113,76) D points with the final engine.
TAG=${1:-dsweep2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 2400 python tools/d_sweep.py 30 512,1024,2048,4096,8192 $OUT/d_sweep_L30.jsonl > $OUT/d_sweep_L30.log 2>&1
ls -la $OUT
