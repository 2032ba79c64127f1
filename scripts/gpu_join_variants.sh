#!/bin/bash
# time the C4 join (probe_diff) with diagnostic library variants, interleaved:
#   bash scripts/gpu_join_variants.sh default alt ...   ("default" = the product library)
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = default ]; then L=$PWD/paper_2512_08365_b200/_lib/libdwb200.so; else L=$PWD/paper_2512_08365_b200/_lib/libdwb200_$v.so; fi
  echo "== $v"; DWB200_LIB=$L timeout 300 python scripts/probe_diff.py C4 4 keys 2>&1 | tail -2
done; done
