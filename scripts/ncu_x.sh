#!/bin/bash
# full ncu capture of one attribution tile-kernel launch (C4 pair side A)
#   bash scripts/ncu_x.sh KIND SUMMATION TAG [kernel-regex]
KIND=${1:-linear}; SUM=${2:-exact}; TAG=${3:-x}; K=${4:-attribute_}
python scripts/probe_attr.py C4 $KIND 3 $SUM > gpurun_out/probe_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
    -o gpurun_out/prof_${TAG} python scripts/probe_attr.py C4 $KIND 2 $SUM > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${TAG}.log; cat gpurun_out/probe_${TAG}.log
