#!/bin/bash
TAG=${1:-knobs76}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for r in 1 2; do
  for kv in "X=0" "SDMRG_ONE_BODY=0" "SDMRG_ONE_BODY=1" "SDMRG_SPLIT=48" "SDMRG_SPLIT=192" "SDMRG_NO_STACK_T=1"; do
    for cfg in "76 4096 113" "30 1024"; do
      echo "[$kv] $cfg: $(env $kv timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)" | sed 's/"lib": "[^"]*", //' | cut -c1-200 >> $OUT/ab.log
    done
  done
done
