#!/bin/bash
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_smem.py -x -q > gpurun_out/pytest_smem.log 2>&1; echo "smem tests rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/pytest_smem.log >> gpurun_out/summary.txt
GERBIL_TRACE=1 timeout 300 python scripts/diag_smem.py 50000000 15 0 0 > /dev/null 2>gpurun_out/trace.log
grep -E "supermer done|histogram|scatter issued|planned|smem count|waves done" gpurun_out/trace.log | tail -7 >> gpurun_out/summary.txt
for M in ${BENCH_MS:-15}; do
timeout 300 python bench.py --m $M --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_m$M.log 2>&1; python scripts/show_bench.py gpurun_out/bench_m$M.log >> gpurun_out/summary.txt 2>&1
done
cat gpurun_out/summary.txt
