#!/bin/bash
# refresh the ncu summaries under profiles/: tile kernel + the join's main kernels (C4)
TAG=${1:-r1}
timeout 900 bash scripts/ncu_tile.sh linear $TAG
python scripts/ncu_summary.py gpurun_out/prof_tiles_C4_linear_$TAG.ncu-rep gpurun_out/tile_$TAG.md 22002823408 > /dev/null 2>&1
timeout 1500 bash scripts/ncu_join.sh $TAG
for k in join_window_findings join_hash_kernel join_pair_bucket join_pair_sub; do
  python scripts/ncu_summary.py gpurun_out/prof_${k}_$TAG.ncu-rep gpurun_out/${k}_$TAG.md > /dev/null 2>&1
done
rm -f gpurun_out/*.ncu-rep
ls gpurun_out/*.md
