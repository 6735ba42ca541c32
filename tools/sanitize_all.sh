#!/bin/bash
# compute-sanitizer over every kernel family (SURVEY §5 race / memory checks):
# memcheck, racecheck (shared-memory hazards) and synccheck on tools/sanitize.py's small
# renders, under each forced scheduler.  -> gpurun_out/sanitize_summary.txt
set -u
mkdir -p gpurun_out
: > gpurun_out/sanitize_summary.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for env in "FRACTAL_SCHED=" "FRACTAL_SCHED=twophase" "FRACTAL_SCHED=refill" \
           "FRACTAL_SCHED=amort" "FRACTAL_SCHED=static" \
           "FRACTAL_SCHED=twophase FRACTAL_P2S=1"; do
  for tool in memcheck racecheck synccheck; do
    log=gpurun_out/sanitize_${tool}_$(echo $env | tr ' =' '__').log
    env $env timeout 1200 $CS --tool $tool --error-exitcode 9 python tools/sanitize.py > $log 2>&1
    rc=$?
    echo "$env $tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)" >> gpurun_out/sanitize_summary.txt
  done
done
cat gpurun_out/sanitize_summary.txt
