#!/bin/bash
# full GPU suite, default bench (C4, e2e, cpu baseline, parity), step launch list
mkdir -p gpurun_out; TAG=${1:-r2c}
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log; tail -4 gpurun_out/pytest_$TAG.log
timeout 1200 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
bash scripts/ncu_step.sh C4 $TAG
python scripts/launch_table.py gpurun_out/launches_step_C4_$TAG.csv | head -40
