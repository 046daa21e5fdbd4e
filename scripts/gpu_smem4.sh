#!/bin/bash
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_smem.py -x -q > gpurun_out/pytest_smem.log 2>&1; echo "smem tests rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/pytest_smem.log >> gpurun_out/summary.txt
for M in 15 13; do
echo "m $M auto bins" >> gpurun_out/summary.txt; GERBIL_TRACE=1 timeout 300 python scripts/diag_smem.py 50000000 $M 0 0 >> gpurun_out/summary.txt 2>gpurun_out/trace.log
grep -E "supermer done|histogram|scatter issued|planned|smem count|waves done" gpurun_out/trace.log | tail -7 >> gpurun_out/summary.txt
done
timeout 300 python bench.py --m 15 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_m15.log 2>&1; python scripts/show_bench.py gpurun_out/bench_m15.log >> gpurun_out/summary.txt 2>&1
if [ "${FULLTESTS:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "all gpu tests rc=$?" >> gpurun_out/summary.txt
  tail -2 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
fi
cat gpurun_out/summary.txt
