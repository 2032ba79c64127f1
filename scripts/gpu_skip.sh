#!/bin/bash
# staging-pipeline speed of diagnostic skip builds (consumers release stages unprocessed)
for v in "$@"; do
  echo "== $v"; DWB200_LIB=paper_2512_08365_b200/_lib/libdwb200_$v.so timeout 120 python scripts/probe_attr.py C4 linear 3 2>&1 | grep "ledger" | tail -1
done
