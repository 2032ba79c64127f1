#!/bin/bash
# diagnosis row: classifier/forced-gap parity, ingest + diff regressions, one short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_diagnose.py tests/test_gpu_ingest.py tests/test_gpu_diff.py tests/test_gpu_shard.py -x -q -m gpu > gpurun_out/diag_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/diag_pytest.log
timeout 300 python scripts/probe_classify.py > gpurun_out/probe_classify.log 2>&1; tail -12 gpurun_out/probe_classify.log
