#!/bin/bash
# Build the FP64-pipe microbenchmark (DMMA vs DFMA issue ceilings).
cd "$(dirname "$0")" && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
