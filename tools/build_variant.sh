#!/bin/bash
# build an experimental library variant: tools/build_variant.sh NAME "-DFLAG=.. ..."
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2305_05581_b200/lib/exp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
  -Xcompiler -fPIC,-fopenmp -lgomp $2 -I include \
  -o paper_2305_05581_b200/lib/exp/lib_$1.so paper_2305_05581_b200/csrc/*.cu
