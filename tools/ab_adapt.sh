mkdir -p gpurun_out/ab1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/ab1/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab1/pytest.log; tail -2 gpurun_out/ab1/pytest.log
for r in 1 2; do
for v in default noadapt; do
  if [ $v = default ]; then unset SDMRG_LIB; else export SDMRG_LIB=paper_2305_05581_b200/lib/exp/lib_$v.so; fi
  for cfg in "30 2048" "50 4096"; do echo "$v $cfg: $(timeout 600 python tools/quick.py $cfg 2>&1 | tail -1)"; done
done; done 2>&1 | tee gpurun_out/ab1/ab.log
