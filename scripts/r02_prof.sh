#!/bin/bash
# ncu --set full captures (source-level) of the named kernels in one bench step: PROF="name:regex:skip ..."
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
ARGS="${BENCH_ARGS:---steps 1 --warmup 3 --no-e2e --no-cpu-baseline}"
for spec in $PROF; do
  IFS=: read name rx skip <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c 1 \
     -o gpurun_out/prof_$name -f python bench.py $ARGS > gpurun_out/ncu_$name.log 2>&1
  echo "$name rc=$?" >> gpurun_out/summary.txt
  ncu -i gpurun_out/prof_$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_$name.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/raw_$name.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep > gpurun_out/details_$name.txt 2>/dev/null
done
cat gpurun_out/summary.txt
