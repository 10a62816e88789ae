#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (every libmds kernel on small problems),
# one tool at a time -> gpurun_out/san_<tool>.txt (+ a one-line summary each)
set -u
OUT=gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
    python tools/sanitize_run.py > $OUT/san_$tool.txt 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run ok' $OUT/san_$tool.txt | tr '\n' ' ')"
done
