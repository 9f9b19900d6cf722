#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every async kernel (tools/sanitize_driver.py).
# Usage (GPU box): bash tools/sanitize.sh [outdir]   -> <outdir>/sanitize_<tool>_<part>.log + summary.txt
OUT=${1:-gpurun_out/sanitize}
mkdir -p $OUT
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
: > $OUT/summary.txt
for tool in memcheck racecheck synccheck; do
  for part in fusion grpo; do
    log=$OUT/sanitize_${tool}_${part}.log
    extra=""
    [ $tool = memcheck ] && extra="--leak-check no"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 1200 $CS --tool $tool $extra --error-exitcode 9 python tools/sanitize_driver.py $part > $log 2>&1
    rc=$?
    echo "$tool $part rc=$rc $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tail -1)" | tee -a $OUT/summary.txt
  done
done
