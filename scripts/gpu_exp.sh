#!/bin/bash
# timings of diagnostic experiment builds (libdwb200_<variant>.so), C4 ledger
for v in "$@"; do
  echo "== $v"; DWB200_LIB=paper_2512_08365_b200/_lib/libdwb200_$v.so timeout 120 python scripts/probe_attr.py C4 ${KIND:-linear} 3 2>&1 | grep "ledger" | tail -1
done
