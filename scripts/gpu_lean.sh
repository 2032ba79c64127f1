#!/bin/bash
# lean exact kernel: parity tests, timing, one ncu capture
mkdir -p gpurun_out; TAG=${1:-lean}
timeout 900 python -m pytest tests/test_gpu_attribution.py tests/test_gpu_scale.py -x -q > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_$TAG.log
timeout 300 python scripts/probe_attr.py C4 linear 4 exact 2>&1 | grep -E "ledger|gen"
timeout 300 python scripts/probe_attr.py C4 step 3 exact 2>&1 | grep -E "ledger"
[ "$2" = "ncu" ] && bash scripts/ncu_x.sh linear exact ${TAG} 'attribute_exact'
exit 0
