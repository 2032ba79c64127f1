#!/bin/bash
# full ncu capture of one attribute_tiles launch (C4, given kind)
KIND=${1:-linear}; TAG=${2:-x}
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:attribute_tiles -s 1 -c 1 \
    -o gpurun_out/prof_tiles_C4_${KIND}_${TAG} python scripts/probe_attr.py C4 $KIND 2 > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
