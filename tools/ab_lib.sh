#!/bin/bash
# A/B library variants on one box (2 rounds, interleaved):
#   tools/ab_lib.sh TAG default twobody ...   (names under lib/exp/lib_NAME.so)
# configs from $CFGS (default "30 2048;50 4096"); GPU tests first unless NOTEST=1
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
fi
IFS=';' read -ra CF <<< "${CFGS:-30 2048;50 4096}"
ORDER=("$@"); REV=(); for ((x=${#ORDER[@]}-1; x>=0; x--)); do REV+=("${ORDER[x]}"); done
for r in 1 2; do
  if [ $r = 1 ]; then LIST=("${ORDER[@]}"); else LIST=("${REV[@]}"); fi  # ABBA: cancels position bias
  for v in "${LIST[@]}"; do
    for cfg in "${CF[@]}"; do
      if [ "$v" = default ]; then res=$(timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)
      else res=$(SDMRG_LIB=paper_2305_05581_b200/lib/exp/lib_$v.so timeout 600 python tools/quick.py $cfg 2>&1 | tail -1); fi
      echo "[$v] $cfg: $res" | sed 's/"lib": "[^"]*", //' | cut -c1-230
    done
  done
done 2>&1 | tee $OUT/ab.log
