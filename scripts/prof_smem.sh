#!/bin/bash
# ncu full capture of the shared-memory count kernel (3rd call of diag_smem: C1 size, m=$M)
set -u
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:count_smem -s 2 -c 1 -o gpurun_out/${OUT:-prof_smem} python scripts/diag_smem.py 50000000 ${M:-15} > gpurun_out/ncu_smem.log 2>&1
echo rc=$?
