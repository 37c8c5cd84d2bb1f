#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_workload.py (GPU box): memcheck,
# racecheck (shared memory), synccheck (barriers, incl. the persistent
# loop's), initcheck.  Summaries -> gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  # racecheck checks shared memory; the Narrow32 kernels have none (and the
  # tool crashes instrumenting them), see tools/sanitize_workload.py
  if [ $tool = racecheck ]; then export PG_SANITIZE_NO_F32=1; else unset PG_SANITIZE_NO_F32; fi
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all \
    --print-limit 50 python tools/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|workload mismatches' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
