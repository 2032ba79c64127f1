#!/bin/bash
for v in "" skip noitems; do
  lib=paper_2512_08365_b200/_lib/libdwb200${v:+_$v}.so
  echo "== variant ${v:-product}"
  DWB200_LIB=$PWD/$lib python scripts/probe_attr.py C4 linear 3 exact 2>&1 | grep ledger | tail -2
done
