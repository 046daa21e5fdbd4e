#!/bin/bash
# bench once per ENVS entry (';'-separated "VAR=val VAR2=val" sets), default build
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
IFS=';' read -ra ES <<< "${ENVS}"
for E in "${ES[@]}"; do
  N=$(echo "$E" | tr -c 'A-Za-z0-9=' '_')
  env $E timeout 300 python bench.py --no-cpu-baseline --steps 3 ${BENCH_ARGS:-} > gpurun_out/bench_$N.log 2>&1; echo "$E rc=$?" >> gpurun_out/summary.txt
done
cat gpurun_out/summary.txt
