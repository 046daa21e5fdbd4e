#!/bin/bash
# Generic round-2 gpurun wrapper: build, then run the commands given in $CMDS (one per line),
# each logged to gpurun_out/cmdN.log; a summary with exit codes and durations at the end.
set -u
mkdir -p gpurun_out
{ nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"; free -g | head -2;
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/host.txt 2>&1
python build_native.py > gpurun_out/build.log 2>&1 || { echo build failed; tail -30 gpurun_out/build.log; exit 1; }
i=0
while IFS= read -r c; do
  [ -z "$c" ] && continue
  i=$((i+1))
  echo "== [$i] $c" >> gpurun_out/summary.txt
  s=$(date +%s)
  bash -c "$c" > gpurun_out/cmd$i.log 2>&1; rc=$?
  echo "   rc=$rc  $(( $(date +%s) - s )) s" >> gpurun_out/summary.txt
  tail -4 gpurun_out/cmd$i.log | cut -c1-400 | sed 's/^/   /' >> gpurun_out/summary.txt
done <<< "$CMDS"
cat gpurun_out/host.txt gpurun_out/summary.txt
