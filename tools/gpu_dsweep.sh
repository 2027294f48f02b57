#!/bin/bash
# D sweep (configs[4]) + GPU tests + default bench line on one box
TAG=${1:-dsweep}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err; tail -c 600 $OUT/bench.json
timeout 1800 python tools/d_sweep.py 30 512,1024,2048,4096,8192 $OUT/d_sweep.jsonl > $OUT/d_sweep.log 2>&1
cat $OUT/d_sweep.jsonl | cut -c1-300
