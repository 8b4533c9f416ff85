#!/bin/bash
# compute-sanitizer over every CUDA path at config T; logs to profiles/r02/.
out=${1:-profiles/r02}
mkdir -p "$out"
for tool in memcheck racecheck initcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_T.py \
      > "$out/sanitizer_$tool.txt" 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$out/sanitizer_$tool.txt" | tail -1)"
done
