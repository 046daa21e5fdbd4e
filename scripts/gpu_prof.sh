#!/bin/bash
# ncu captures of the hot kernels + a launch list of one bench step.
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
ARGS="--reads ${BENCH_READS:-5000000} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
prof() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
     -o gpurun_out/prof_$1 python bench.py $ARGS > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/summary.txt
}
prof count 'count_kernel' ${SKIP_COUNT:-300}
prof supermer 'supermer_kernel' 3
prof compact 'compact_kernel' ${SKIP_COUNT:-300}
if [ "${LAUNCHES:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?" >> gpurun_out/summary.txt
fi
cat gpurun_out/summary.txt
