#!/bin/bash
# One gpurun call: GPU parity tests, the bench line, the ncu launch list and
# one full ncu capture of the top kernel.  Usage: tools/gpu_round.sh TAG
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --scale "" > $OUT/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -s 3 -c 1 \
    -o $OUT/prof python tools/prof_apply.py 30 2048 2 > $OUT/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm -s 2 -c 1 \
    -o $OUT/prof_p1 python tools/prof_apply.py 30 2048 2 > $OUT/ncu_p1.log 2>&1
ls -la $OUT
