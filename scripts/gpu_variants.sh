#!/bin/bash
# time the exact ledger (C4 linear) with several diagnostic builds, interleaved
for rep in 1 2; do
for v in "$@"; do
  echo "== $v"; DWB200_LIB=$PWD/paper_2512_08365_b200/_lib/libdwb200_$v.so timeout 300 python scripts/probe_attr.py C4 linear 3 exact 2>&1 | grep ledger | tail -1
done; done
