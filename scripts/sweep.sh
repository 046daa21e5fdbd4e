#!/bin/bash
# tuning sweep on the full C1 bench (device-timed value only)
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
for T in ${TABLES:-96 128 192 384}; do
  GERBIL_COUNT_U=${U:-1} timeout 200 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --table-mb $T > gpurun_out/sweep_U${U:-1}_T${T}.log 2>&1
  echo "T=$T rc=$?" >> gpurun_out/summary.txt
done
if [ -n "${NCU_K:-}" ]; then
GERBIL_COUNT_U=${U:-1} timeout 400 ncu --set full --clock-control none --import-source on -k regex:$NCU_K -s ${NCU_S:-100} -c 1 \
   -o gpurun_out/prof_iter python bench.py --reads 5000000 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --table-mb ${NCU_T:-96} > gpurun_out/ncu_iter.log 2>&1
echo "ncu rc=$?" >> gpurun_out/summary.txt
fi
cat gpurun_out/summary.txt
