#!/bin/bash
# exact tile kernel: variants (product / staging only / pass B only) + one ncu --set full capture
mkdir -p gpurun_out
bash scripts/gpu_x3.sh > gpurun_out/x3_r2b.log 2>&1
cat gpurun_out/x3_r2b.log
python scripts/probe_attr.py C4 linear 3 reference 2>&1 | grep ledger | tail -1
bash scripts/ncu_x.sh linear exact r2b_exact 'attribute_exact'
