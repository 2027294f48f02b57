#!/bin/bash
# Iteration call: GPU parity tests + per-phase timing at bench scale.
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
shift
for cfg in "${@:-30 2048}"; do
  timeout 600 python tools/quick.py $cfg 2>&1 | tail -2 | tee -a $OUT/quick.log
done
