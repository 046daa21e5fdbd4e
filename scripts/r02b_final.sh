#!/bin/bash
# Round-2 final evidence in one GPU call (after the reference-table and step-(b) changes of the
# second half): benches (C1 default + reference arm + C2..C4), the ncu launch list of a C1 step,
# ncu --set full captures of the hot kernels (C1 and C4) exported to CSV, compute-sanitizer.
set -u
mkdir -p gpurun_out
python build_native.py > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
{ nproc; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,clocks.max.sm --format=csv; } > gpurun_out/host.txt 2>&1
run() { echo "== $1" >> gpurun_out/summary.txt; s=$(date +%s); bash -c "$2"; echo "   rc=$? $(( $(date +%s) - s )) s" >> gpurun_out/summary.txt; }
if [ "${TESTS:-1}" = "1" ]; then
run gpu_tests "timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r02_gpu_tests.txt 2>&1"
fi
if [ "${BENCH:-1}" = "1" ]; then
run bench_c1 "timeout 1200 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err"
run bench_ref "timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err"
for c in C2 C3k65 C3k100 C4; do
  run bench_$c "timeout 900 python bench.py --config $c --no-e2e --no-cpu-full > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err"
done
fi
if [ "${LAUNCH:-1}" = "1" ]; then
run launches "timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1"
fi
if [ "${NCU:-1}" = "1" ]; then
# count_ref_kernel: the tier-1 launch of the first call (~90 % of the tier time; a --set full replay
# of all 16 launches of a call saves and restores tens of GB per pass: > 30 min)
nref=$(python -c "import json;print(json.load(open('gpurun_out/r02_bench_C4.json'))['roofline']['launches_per_step'])" 2>/dev/null || echo 16)
for spec in ${PROF:-c1_supermer:C1:supermer_kernel:3:1:3 c1_smem:C1:count_smem_kernel:0:8:3 c1_part:C1:partition64:0:8:3 c1_regroup:C1:regroup_counted:3:1:3 c1_ghist:C1:group_hist:3:1:3 c4_ref:C4:count_ref_kernel:0:1:0 c4_supermer:C4:supermer_kernel:3:1:3}; do
  IFS=: read name cfg rx skip cnt wu <<< "$spec"
  run ncu_$name "timeout 1800 ncu --set full --clock-control none --import-source on -k regex:$rx -s $skip -c $cnt -o gpurun_out/prof_$name -f python bench.py --config $cfg --steps 1 --warmup $wu --no-e2e --no-cpu-baseline > gpurun_out/ncu_$name.log 2>&1"
  ncu -i gpurun_out/prof_$name.ncu-rep --page raw --csv > gpurun_out/raw_$name.csv 2>/dev/null
  ncu -i gpurun_out/prof_$name.ncu-rep > gpurun_out/details_$name.txt 2>/dev/null
  python scripts/ncu_srcprof.py gpurun_out/prof_$name.ncu-rep 60 > gpurun_out/src_$name.txt 2>/dev/null
  rm -f gpurun_out/prof_$name.ncu-rep  # the merge-back limit is 64 MiB: keep the exports only
done
fi
# compute-sanitizer is closed on this pool (runs under it left GPUs needing a reset): off by default
if [ "${SAN:-0}" = "1" ]; then
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
  run san_$tool "timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 --kernel-name-exclude kns=synth python scripts/sanitize_cases.py ${CASES:-smem_k40 smem_alla ref_k150 ref_alla ref_k200_zfp l2_k40} > gpurun_out/sanitize_$tool.log 2>&1"
done
fi
cat gpurun_out/summary.txt
