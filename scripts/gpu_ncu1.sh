#!/bin/bash
# one ncu --set full capture: KERNEL regex, SKIP launches, OUT name; bench on 5e6 reads
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$KERNEL -s ${SKIP:-3} -c 1 \
  -o gpurun_out/$OUT python bench.py --reads ${READS:-5000000} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$OUT.log 2>&1
echo "ncu rc=$?"
