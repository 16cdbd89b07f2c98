#!/usr/bin/env bash
# compute-sanitizer over scripts/sanitize_cases.py; summaries to gpurun_out/sanitize_<tool>.log
set -u
mkdir -p gpurun_out
python scripts/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/sanitize_plain.log; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python scripts/sanitize_cases.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -4 gpurun_out/sanitize_$tool.log
done
