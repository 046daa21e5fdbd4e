#!/bin/bash
# One gpurun session: smoke, gpu tests, bench. Logs to gpurun_out/.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python build_native.py > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
timeout 600 python bench.py --reads ${BENCH_READS:-5000000} --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1; echo "bench_small rc=$?" >> gpurun_out/summary.txt
if [ "${FULL:-0}" = "1" ]; then
  timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
fi
tail -3 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
