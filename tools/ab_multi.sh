#!/bin/bash
# A/B several plan-build env settings on one box (2 rounds, interleaved):
#   tools/ab_multi.sh TAG "none" "SDMRG_X=1" "SDMRG_X=2 SDMRG_Y=1" ...
# configs from $CFGS (default "30 2048;50 4096")
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
IFS=';' read -ra CF <<< "${CFGS:-30 2048;50 4096}"
ORDER=("$@"); REV=(); for ((x=${#ORDER[@]}-1; x>=0; x--)); do REV+=("${ORDER[x]}"); done
for r in 1 2; do
  if [ $r = 1 ]; then LIST=("${ORDER[@]}"); else LIST=("${REV[@]}"); fi  # ABBA: cancels position bias
  for knob in "${LIST[@]}"; do
    for cfg in "${CF[@]}"; do
      if [ "$knob" = none ]; then res=$(timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)
      else res=$(env $knob timeout 600 python tools/quick.py $cfg 2>&1 | tail -1); fi
      echo "[$knob] $cfg: $res" | cut -c1-260
    done
  done
done 2>&1 | tee $OUT/ab.log
