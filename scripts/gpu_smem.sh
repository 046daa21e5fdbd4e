#!/bin/bash
# shared-memory count path: parity tests + C1 bench at m=13 (auto) vs m=7
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_smem.py -x -q > gpurun_out/pytest_smem.log 2>&1; echo "smem tests rc=$?" >> gpurun_out/summary.txt
tail -3 gpurun_out/pytest_smem.log >> gpurun_out/summary.txt
for M in ${BENCH_MS:-13 12 15}; do
  timeout 300 python bench.py --m $M --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_m$M.log 2>&1; echo "bench m=$M rc=$?" >> gpurun_out/summary.txt
  python scripts/show_bench.py gpurun_out/bench_m$M.log >> gpurun_out/summary.txt 2>&1
done
cat gpurun_out/summary.txt
