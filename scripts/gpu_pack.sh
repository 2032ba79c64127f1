#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_packed.py tests/test_gpu_diagnose.py tests/test_gpu_ingest.py tests/test_gpu_shard.py -x -q > gpurun_out/pack_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pack_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/pack_bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/pack_bench.log
