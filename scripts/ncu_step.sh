#!/bin/bash
# launch list of one full bench step (the second of two), all of our + CUB kernels
CFG=${1:-C4}; TAG=${2:-r1}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base mangled -k regex:'_ZN2dw|_ZN3cub' --csv \
    --log-file gpurun_out/launches_step_${CFG}_${TAG}.csv python scripts/probe_step.py $CFG 2 > gpurun_out/ncu_step.log 2>&1
tail -2 gpurun_out/ncu_step.log
