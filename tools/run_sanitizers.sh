#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py), logs under $1
out=${1:-gpurun_out/sanitizer}
mkdir -p "$out"
for tool in memcheck racecheck synccheck; do
  for c in stage clsjit segment gemm64 gemm256 gemm256_1cta klt fixed fixed_row corr; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_cases.py $c > "$out/${tool}_${c}.log" 2>&1
    echo "$tool $c rc=$?" | tee -a "$out/summary.txt"
  done
done
