#!/bin/bash
# shared-memory count kernel ncu capture (C1, m=15, auto bins) + regroup kernel + bench line
set -u
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"count_smem|regroup_fine" -s 4 -c 2 -o gpurun_out/prof_smem4 python scripts/diag_smem.py 50000000 15 0 0 > gpurun_out/ncu_smem.log 2>&1
echo ncu rc=$?
timeout 300 python bench.py --m 15 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_m15.log 2>&1; python scripts/show_bench.py gpurun_out/bench_m15.log
