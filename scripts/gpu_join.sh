#!/bin/bash
# join parity + timing (+ optional launch list of one diff)
mkdir -p gpurun_out; TAG=${1:-join}
timeout 900 python -m pytest tests/test_gpu_diff.py tests/test_gpu_scale.py tests/test_gpu_shard.py tests/test_gpu_diagnose.py -x -q > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_$TAG.log
timeout 300 python scripts/probe_diff.py C4 4 keys 2>&1 | tail -3
if [ "$2" = "ncu" ]; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base mangled -k regex:'_ZN2dw|_ZN3cub' --csv --log-file gpurun_out/launches_$TAG.csv \
    python scripts/probe_diff.py C4 2 keys > gpurun_out/ncu_$TAG.log 2>&1
  python scripts/launch_table.py gpurun_out/launches_$TAG.csv | head -30
fi
exit 0
