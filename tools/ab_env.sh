#!/bin/bash
# A/B one plan-build env knob on one box: tools/ab_env.sh TAG "ENV=VAL" [cfg ...]
TAG=$1; KNOB=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log; tail -2 $OUT/pytest.log
for r in 1 2; do
  for v in default knob; do
    for cfg in "${@:-30 2048}"; do
      if [ $v = default ]; then res=$(timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)
      else res=$(env $KNOB timeout 600 python tools/quick.py $cfg 2>&1 | tail -1); fi
      echo "$v $cfg: $res"
    done
  done
done 2>&1 | tee $OUT/ab.log
