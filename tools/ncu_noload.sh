OUT=gpurun_out/nl; mkdir -p $OUT
SDMRG_LIB=paper_2305_05581_b200/lib/exp/lib_noload.so python tools/quick.py 30 2048 | tail -1
SDMRG_LIB=paper_2305_05581_b200/lib/exp/lib_noload.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:seg_gemm_kernel -s 3 -c 1 -o $OUT/prof_p2 python tools/prof_apply.py 30 2048 2 > $OUT/ncu.log 2>&1
tail -1 $OUT/ncu.log
