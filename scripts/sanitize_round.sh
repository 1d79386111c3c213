#!/bin/bash
# compute-sanitizer over the small workloads of scripts/sanitize_case.py.
set -u
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
for tool in memcheck racecheck synccheck initcheck; do
  for c in flat_golden flat_c1 ivf_golden encoder_small; do
    timeout 420 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_case.py $c \
      > "$OUT/sanitize_${tool}_${c}.log" 2>&1
    echo "$tool $c rc=$?" | tee -a "$OUT/sanitize_summary.txt"
  done
done
