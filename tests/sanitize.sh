#!/usr/bin/env bash
# compute-sanitizer over every kernel family (scripts/sanitize_cases.py);
# one log per tool under ${1:-gpurun_out/sanitizer}.  Run on a GPU box.
OUT=${1:-gpurun_out/sanitizer}
mkdir -p "$OUT"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  timeout 1800 compute-sanitizer --tool $tool $extra --error-exitcode 9 \
    python scripts/sanitize_cases.py > "$OUT/$tool.txt" 2>&1
  echo "$tool rc=$?" | tee -a "$OUT/summary.txt"
  tail -3 "$OUT/$tool.txt" >> "$OUT/summary.txt"
done
