#!/bin/bash
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
timeout 400 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -2 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
timeout 900 python -m pytest tests/test_gpu_zfullsize.py -x -q -m gpu -s > gpurun_out/pytest_full.log 2>&1; echo "full rc=$?" >> gpurun_out/summary.txt
tail -2 gpurun_out/pytest_full.log >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
