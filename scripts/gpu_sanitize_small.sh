#!/bin/bash
# compute-sanitizer, every tool, over the small workload only (scripts/sanitize.py)
mkdir -p gpurun_out; TAG=${1:-s}
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 python scripts/sanitize.py > gpurun_out/sanitize_${t}_$TAG.log 2>&1
  echo "$t rc=$?"; tail -1 gpurun_out/sanitize_${t}_$TAG.log
done
