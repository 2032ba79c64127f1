#!/bin/bash
# round-2 status run: full GPU suite, default bench, step launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r2a.txt 2>&1
nproc >> gpurun_out/smi_r2a.txt; lscpu | grep "Model name" >> gpurun_out/smi_r2a.txt
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 > gpurun_out/pytest_r2a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r2a.log; tail -40 gpurun_out/pytest_r2a.log
timeout 900 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
echo "bench rc=$?"; cat gpurun_out/bench_r2a.json; tail -5 gpurun_out/bench_r2a.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r2a.csv python bench.py --steps 1 --warmup 1 --no-e2e > gpurun_out/ncu_bench_r2a.log 2>&1
echo "ncu rc=$?"
