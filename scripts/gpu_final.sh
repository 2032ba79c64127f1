#!/bin/bash
# end-of-round checks on one B200: GPU tests, smoke, bench (ours + reference arm),
# the time-window path under torchrun (2 ranks sharing the GPU over gloo)
TAG=${1:-final}
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err; echo "ref rc=$?"; tail -c 400 gpurun_out/bench_ref_${TAG}.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --shard window --dist-backend gloo --config C2 --steps 2 --warmup 1 > gpurun_out/bench_window_${TAG}.json 2> gpurun_out/bench_window_${TAG}.err; echo "window rc=$?"
tail -c 300 gpurun_out/bench_window_${TAG}.json
