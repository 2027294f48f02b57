#!/bin/bash
# Round-end GPU pass: smoke, the whole -m gpu suite, the bench line and the
# reference arm, the ncu launch list of the bench command, one full ncu
# capture of each engine kernel at the bench workload (L=50 D=4096).  tools/gpu_final.sh TAG
TAG=${1:-final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
if [ "$2" != "skip-tests" ]; then
  timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
timeout 1200 python bench.py --steps 10 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --scale "" --sweep "" > $OUT/bench_under_ncu.log 2>&1
for k in "p1:sdmrg::seg_gemm_kernel<.bool.0, .bool.1" "p2small:sdmrg::seg_gemm_kernel<.bool.0, .bool.0" "p2big:sdmrg_big::seg_gemm_kernel<.bool.0, .bool.0"; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k regex:"${k#*:}" -s 0 -c 1 -o $OUT/prof_${k%%:*} python tools/prof_apply.py 50 4096 1 > $OUT/ncu_${k%%:*}.log 2>&1
done
ls -la $OUT
