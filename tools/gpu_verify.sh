#!/bin/bash
# The pruned engine: the whole GPU suite, smoke, and an ABBA timing against
# the pre-prune build (lib/exp/lib_preprune.so).
TAG=${1:-verify}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
P=paper_2305_05581_b200/lib/exp/lib_preprune.so
for order in "new old" "old new"; do
  for v in $order; do
    for cfg in "50 4096" "30 2048"; do
      if [ $v = new ]; then L=""; else L=$P; fi
      echo "[$v] $cfg: $(SDMRG_LIB=$L timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)" | sed 's/"lib": "[^"]*", //' | cut -c1-200 >> $OUT/ab.log
    done
  done
done
ls -la $OUT
