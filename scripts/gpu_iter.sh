#!/bin/bash
# quick iteration: gpu tests, small+full bench, optional ncu of one kernel
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -2 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
timeout 240 python bench.py --reads 5000000 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_small.log 2>&1; echo "bench_small rc=$?" >> gpurun_out/summary.txt
if [ "${FULL:-1}" = "1" ]; then
timeout 400 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
fi
if [ -n "${NCU_K:-}" ]; then
timeout 400 ncu --set full --clock-control none --import-source on -k regex:$NCU_K -s ${NCU_S:-100} -c 1 \
   -o gpurun_out/prof_iter python bench.py --reads 5000000 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_iter.log 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
fi
cat gpurun_out/summary.txt
