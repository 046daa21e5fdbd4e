#!/bin/bash
# Round profiling evidence: launch list of bench steps + ncu full captures (full C1 config).
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?" >> gpurun_out/summary.txt
cap() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:$2 -s $3 -c 1 \
     -o gpurun_out/prof_$1 python bench.py $ARGS > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/summary.txt
}
# warm-up 3 steps then the timed step: count/compact launches per step ~ waves (~150)
cap count count_inline ${SKIP_COUNT:-500}
cap compact compact_inline ${SKIP_COUNT:-500}
cap supermer supermer_kernel 3
cap scatter scatter_smem 3
cat gpurun_out/summary.txt
