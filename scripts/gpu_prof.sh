#!/bin/bash
# ncu captures of the three hot kernels + a launch list of one bench step.
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
ARGS="--reads ${BENCH_READS:-5000000} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
for k in count_kernel compact_kernel supermer_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-20} -c 1 \
     -o gpurun_out/prof_$k python bench.py $ARGS > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?" >> gpurun_out/summary.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?" >> gpurun_out/summary.txt
cat gpurun_out/summary.txt
