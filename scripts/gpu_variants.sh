#!/bin/bash
# time the exact ledger (C4 linear) with several diagnostic builds, interleaved
#   bash scripts/gpu_variants.sh default v1 v2 ...   ("default" = the product library)
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = default ]; then L=$PWD/paper_2512_08365_b200/_lib/libdwb200.so; else L=$PWD/paper_2512_08365_b200/_lib/libdwb200_$v.so; fi
  echo "== $v"; DWB200_LIB=$L timeout 300 python scripts/probe_attr.py C4 linear 3 exact 2>&1 | grep -E "ledger|Error|error" | tail -1
done; done
