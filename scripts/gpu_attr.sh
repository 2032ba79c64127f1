#!/bin/bash
# attribution parity (GPU tests) + C4 exact ledger timing + kernel time (ncu launch list)
mkdir -p gpurun_out; TAG=${1:-attr}
timeout 900 python -m pytest tests/test_gpu_attribution.py tests/test_gpu_scale.py -x -q > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_$TAG.log
for k in linear step; do timeout 300 python scripts/probe_attr.py C4 $k 4 exact 2>&1 | grep ledger | tail -2; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attribute_exact --csv python scripts/probe_attr.py C4 linear 2 exact 2>/dev/null | grep -o '"[0-9]*"$'
