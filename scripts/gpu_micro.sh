#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_micro scripts/l2_micro.cu
for T in 32 48 64; do timeout 60 /tmp/l2_micro $T 8; done > gpurun_out/l2_micro.txt 2>&1
cat gpurun_out/l2_micro.txt
