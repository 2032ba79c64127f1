#!/bin/bash
# one ncu --set full capture of a kernel (regex) inside a probe command
#   bash scripts/ncu_kern.sh TAG REGEX python scripts/probe_diff.py C4 2 keys
TAG=$1; K=$2; shift 2
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_${TAG} "$@" > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log
