#!/bin/bash
# End-of-round call: the round script + the D sweep + the reference arm line
TAG=${1:-final}
bash tools/gpu_round.sh $TAG
OUT=gpurun_out/$TAG
timeout 1200 python tools/d_sweep.py 30 512,1024,2048,4096,8192 $OUT/d_sweep.jsonl > $OUT/d_sweep.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
tail -c 400 $OUT/bench_reference.json
