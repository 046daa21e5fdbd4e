#!/bin/bash
# Round evidence (after the shared-memory count path): GPU tests, bench (full C1, e2e, cpu baseline),
# reference arm, launch list of one timed step, ncu full captures of the step's kernels.
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
export PYTHONPATH=$PWD
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/summary.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/summary.txt
tail -1 gpurun_out/pytest_gpu.log >> gpurun_out/summary.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/summary.txt
python scripts/show_bench.py gpurun_out/bench.log >> gpurun_out/summary.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/summary.txt
ARGS="--steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py $ARGS > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?" >> gpurun_out/summary.txt
cap() {  # name regex skip [count]
  timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:$2 -s $3 -c ${4:-1} \
     -o gpurun_out/prof_$1 python bench.py $ARGS > gpurun_out/ncu_$1.log 2>&1
  echo "$1 rc=$?" >> gpurun_out/summary.txt
}
# 3 warm-up steps x 2 shared-memory launches (tiers 1 and 2): the timed step's pair
cap smem count_smem 6 2
cap supermer supermer_kernel 3
cap regroup regroup_fine 3
cap scatter scatter_smem 3
cat gpurun_out/summary.txt
