#!/bin/bash
# one GPU session: parity tests, smoke, bench line, launch list, full capture of the tile kernel
TAG=${1:-r1}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
cat gpurun_out/bench_${TAG}.json
[ "$2" = "noprof" ] && exit 0
timeout 900 bash scripts/ncu_step.sh C4 ${TAG}
timeout 900 bash scripts/ncu_attr.sh C4 step ${TAG}
ls -la gpurun_out
