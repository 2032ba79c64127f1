#!/bin/bash
# round artefacts: bench line (default config, with e2e), launch list of one step, full capture of the tile kernel
TAG=${1:-r1}
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
tail -c 600 gpurun_out/bench_${TAG}.json
timeout 900 bash scripts/ncu_step.sh C4 ${TAG}
timeout 900 bash scripts/ncu_tile.sh linear ${TAG}
