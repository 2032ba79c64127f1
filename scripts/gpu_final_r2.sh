#!/bin/bash
# round-2 evidence: GPU tests, smoke, default bench (C4, e2e, cpu baseline,
# parity), C5 corpus bench, the step's launch list, ncu captures of the tile
# kernel and the join kernels
mkdir -p gpurun_out; TAG=${1:-r2z}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 1500 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err; echo "c5 rc=$?"
bash scripts/ncu_step.sh C4 $TAG
bash scripts/ncu_x.sh linear exact ${TAG}_tile attribute_exact
for k in jb_pass_kernel jb_hash_kernel jb_bucket_kernel join_window_findings_kernel join_pair_sub_kernel; do
  bash scripts/ncu_kern.sh ${TAG}_$k $k timeout 900 python scripts/probe_diff.py C4 2 deltas
done
