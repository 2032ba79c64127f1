#!/bin/bash
# phase-timer build: cycles per tile phase at C4 (diagnostic; timings under it are not bench values)
DWB200_LIB=paper_2512_08365_b200/_lib/libdwb200_prof.so timeout 300 python scripts/probe_attr.py C4 ${1:-linear} 2 2>&1 | tail -14
DWB200_LIB=paper_2512_08365_b200/_lib/libdwb200_skip.so timeout 300 python scripts/probe_attr.py C4 ${1:-linear} 3 2>&1 | grep "ledger" | tail -2
