#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py, one tool per run, logs in gpurun_out/$TAG/.
#   bash tools/sanitize.sh TAG "memcheck:case,case racecheck:case synccheck:case ..."
set -u
TAG=$1; SPECS=$2
OUT=gpurun_out/$TAG; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for spec in $SPECS; do
  tool=${spec%%:*}; cases=${spec#*:}; cases=${cases//,/ }
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
    python tools/sanitize_cases.py $cases > $OUT/sanitize_$tool.log 2>&1
  rc=$?
  echo "$tool ($cases): rc=$rc; $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $OUT/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
