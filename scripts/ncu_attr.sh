#!/bin/bash
# per-kernel launch list for one C4 ledger (after warm-up), then a full capture of the tile kernel
CFG=${1:-C4}; KIND=${2:-step}; TAG=${3:-r1}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --kernel-name-base mangled -k regex:'_ZN2dw|_ZN3cub' -s 10 -c 10 --csv \
    --log-file gpurun_out/launches_${CFG}_${KIND}_${TAG}.csv python scripts/probe_attr.py $CFG $KIND 2 > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:attribute_tiles -s 1 -c 1 \
    -o gpurun_out/prof_tiles_${CFG}_${KIND}_${TAG} python scripts/probe_attr.py $CFG $KIND 2 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
