#!/bin/bash
# compute-sanitizer over the step's kernels: the small workload (every tool),
# then racecheck / synccheck at a size whose tile loop wraps the 8-stage TMA
# ring several times per CTA (300k ops, 3M samples per trace: ~20 tiles per CTA)
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python scripts/sanitize.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; tail -1 gpurun_out/sanitize_$t.log
done
for t in racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $t --print-limit 50 python scripts/sanitize.py 300000 > gpurun_out/sanitize_${t}_300k.log 2>&1
  echo "$t 300k rc=$?"; tail -1 gpurun_out/sanitize_${t}_300k.log
done
