#!/bin/bash
# round-2 closing evidence after the late changes: GPU tests, smoke, default bench (C4),
# the reference arm, C5 corpus, C2 / C3 / C3-split, the step's launch list,
# an ncu capture of the tile kernel and of the waste-sum pass
mkdir -p gpurun_out; TAG=${1:-r2j}
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 1500 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 1500 python bench.py --config C5 --steps 3 --warmup 3 > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err; echo "c5 rc=$?"
for c in C2 C3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_${c}_$TAG.json 2> gpurun_out/bench_${c}_$TAG.err; echo "$c rc=$?"; done
timeout 900 python bench.py --config C3 --overlap split --steps 10 --warmup 3 > gpurun_out/bench_C3s_$TAG.json 2> gpurun_out/bench_C3s_$TAG.err; echo "C3s rc=$?"
bash scripts/ncu_step.sh C4 $TAG
bash scripts/ncu_x.sh linear exact ${TAG}_tile attribute_exact
for k in waste_sum_kernel fx_sum_kernel; do
  bash scripts/ncu_kern.sh ${TAG}_$k $k timeout 900 python scripts/probe_diff.py C4 2 deltas
done
