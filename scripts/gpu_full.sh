#!/bin/bash
set -u
mkdir -p gpurun_out
{ nproc; free -g; nvidia-smi --query-gpu=name,memory.total --format=csv; } > gpurun_out/box.txt 2>&1
python build_native.py > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_zfullsize.py -x -q -m gpu -s > gpurun_out/pytest_full.log 2>&1; echo "full rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
