#!/bin/bash
# Copy one r02b_final.sh evidence directory into profiles/ (benches, launch list, ncu summaries,
# roofline_traffic.json):  bash scripts/r02_collect.sh gpurun_out
set -eu
shopt -s nullglob
src=${1:-gpurun_out}
for f in "$src"/r02_bench*.json; do cp "$f" profiles/; done
[ -s "$src/r02_gpu_tests.txt" ] && { echo "# r02: python -m pytest tests -m gpu on one B200 (scripts/r02b_final.sh)"; tail -22 "$src/r02_gpu_tests.txt"; } > profiles/r02_gpu_tests.txt
if [ -s "$src/r02_launches.csv" ]; then
  { echo "# r02 ncu launch list of one timed C1 step (bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline; ncu --metrics gpu__time_duration.sum --clock-control none: cold, serialised)";
    python scripts/launch_summary.py "$src/r02_launches.csv"; } > profiles/r02_launches.txt
fi
python scripts/roofline_traffic.py "$src" profiles/r02 > /dev/null
for d in "$src"/details_*.txt; do
  name=$(basename "$d" .txt); name=${name#details_}
  { echo "# r02: ncu --set full --clock-control none --import-source on (scripts/r02b_final.sh), kernel regex of capture $name";
    grep -E "^\s+(void|gerbil|[a-z_]+::)|Section:|Duration|Throughput|Ipc|Issue Slots|Hit Rate|Warp Cycles|Occupancy|Registers|Shared Memory|Block Size|Grid Size|Executed Instructions|Active Threads" "$d" | grep -v "^\s*$";
    if [ -s "$src/src_$name.txt" ]; then echo "# source lines by warp-stall samples (scripts/ncu_srcprof.py)"; sed -n '1,31p' "$src/src_$name.txt"; fi; } > "profiles/r02_ncu_$name.txt"
done
ls -la profiles/ | tail -40
