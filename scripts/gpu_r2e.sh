#!/bin/bash
# reference tests through the shim, sanitizers on the small step workload,
# ncu captures of the join kernels
mkdir -p gpurun_out
bash scripts/ref_tests_shim.sh run
python scripts/sanitize.py > gpurun_out/sanitize_plain.log 2>&1; tail -2 gpurun_out/sanitize_plain.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 50 python scripts/sanitize.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; tail -3 gpurun_out/sanitize_$t.log
done
for k in jb_hash_kernel jb_bucket_kernel join_window_findings_kernel join_pair_sub_kernel; do
  bash scripts/ncu_kern.sh r2n_$k $k timeout 900 python scripts/probe_diff.py C4 2 keys
done
