#!/bin/bash
# build + bench each VARIANTS entry (nvcc -D flags, ';'-separated), then rebuild the default
set -u
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS}"
for V in "${VS[@]}"; do
  N=$(echo "$V" | tr -c 'A-Za-z0-9=' '_')
  GERBIL_NVCC_EXTRA="$V" python build_native.py > gpurun_out/build_$N.log 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 ${BENCH_ARGS:-} > gpurun_out/bench_$N.log 2>&1; echo "$V rc=$?" >> gpurun_out/summary.txt
done
python build_native.py --force > gpurun_out/build.log 2>&1
if [ "${TESTS:-1}" = "1" ]; then
timeout 400 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
fi
cat gpurun_out/summary.txt
