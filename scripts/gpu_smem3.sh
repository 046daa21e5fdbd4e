#!/bin/bash
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_smem.py -x -q > gpurun_out/pytest_smem.log 2>&1; echo "smem tests rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/pytest_smem.log >> gpurun_out/summary.txt
echo "m 15" >> gpurun_out/summary.txt; GERBIL_TRACE=1 timeout 300 python scripts/diag_smem.py 50000000 15 0 >> gpurun_out/summary.txt 2>gpurun_out/trace.log
grep -E "call|smem|supermer|scatter|waves" gpurun_out/trace.log | tail -12 >> gpurun_out/summary.txt
if [ "${FULLTESTS:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "all gpu tests rc=$?" >> gpurun_out/summary.txt
  tail -2 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
fi
cat gpurun_out/summary.txt
