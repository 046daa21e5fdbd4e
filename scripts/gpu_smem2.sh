#!/bin/bash
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_smem.py -x -q > gpurun_out/pytest_smem.log 2>&1; echo "smem tests rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/pytest_smem.log >> gpurun_out/summary.txt
for m in 13 15; do echo "m $m" >> gpurun_out/summary.txt; timeout 300 python scripts/diag_smem.py 50000000 $m 0 >> gpurun_out/summary.txt 2>&1; done
cat gpurun_out/summary.txt
