#!/bin/bash
# full ncu captures of the join kernels (second launch each, C4 probe_diff)
mkdir -p gpurun_out; TAG=${1:-r2j}
for k in jb_pass_kernel jb_hash_kernel jb_bucket_kernel join_window_findings_kernel join_pair_sub_kernel; do
  bash scripts/ncu_kern.sh ${TAG}_$k $k timeout 900 python scripts/probe_diff.py C4 2 keys
done
