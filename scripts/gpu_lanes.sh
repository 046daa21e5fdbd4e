#!/bin/bash
# compare the serial and two-lane wave schedules (full C1 bench), then the GPU tests
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
for L in 1 2; do
  GERBIL_WAVE_LANES=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_l$L.log 2>&1; echo "lanes=$L rc=$?" >> gpurun_out/summary.txt
done
for T in 64 96 192; do
  GERBIL_WAVE_LANES=2 timeout 300 python bench.py --no-cpu-baseline --no-e2e --table-mb $T > gpurun_out/bench_t$T.log 2>&1; echo "t=$T rc=$?" >> gpurun_out/summary.txt
done
timeout 400 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -2 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
