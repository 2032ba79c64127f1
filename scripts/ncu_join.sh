#!/bin/bash
# full ncu captures of the main join kernels (C4 pair), one launch each
TAG=${1:-x}
for k in join_window_findings join_hash_kernel join_pair_bucket join_pair_sub; do
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$k -s 0 -c 1 \
      -o gpurun_out/prof_${k}_${TAG} python scripts/probe_diff.py C4 1 keys > gpurun_out/ncu_${k}_${TAG}.log 2>&1
  tail -1 gpurun_out/ncu_${k}_${TAG}.log
done
