#!/bin/bash
# round-2 GPU session helper: build check, selected tests, a short bench.
#   gpurun -- 'bash scripts/gpu_r2.sh TAG "pytest args" "bench args"'
TAG=${1:-r2}
TESTS=${2:-}
BENCH=${3:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$TAG.txt 2>&1
if [ -n "$TESTS" ]; then
  timeout 1500 python -m pytest $TESTS -x -q > gpurun_out/pytest_$TAG.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
  tail -5 gpurun_out/pytest_$TAG.log
fi
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py $BENCH > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
  echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json; tail -5 gpurun_out/bench_$TAG.err
fi
