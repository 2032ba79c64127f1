#!/bin/bash
# full ncu captures of the step's top kernels (one launch each): exact tile
# kernel (C4 linear) and the join kernels (C4 probe_diff)
mkdir -p gpurun_out; TAG=${1:-r2n}
bash scripts/ncu_x.sh linear exact ${TAG}_tile attribute_exact
for k in jb_pass_kernel jb_hash_kernel jb_bucket_kernel join_window_findings_kernel; do
  bash scripts/ncu_kern.sh ${TAG}_$k $k timeout 900 python scripts/probe_diff.py C4 1 keys
done
ls -la gpurun_out
