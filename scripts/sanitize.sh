#!/bin/bash
# compute-sanitizer over scripts/sanitize_cases.py: memcheck, racecheck, synccheck, initcheck.
# Summaries land in gpurun_out/sanitize_<tool>.log (copied to profiles/ for the record).
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 --kernel-name-exclude kns=synth \
     python scripts/sanitize_cases.py ${CASES:-smem_k40 smem_k65_mc2 smem_alla ref_k150 ref_alla l2_k28 l2_k40 l2_k200} > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/summary.txt
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/summary.txt
done
cat gpurun_out/summary.txt
