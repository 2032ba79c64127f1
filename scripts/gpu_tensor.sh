#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tensor.py tests/test_gpu_diagnose.py tests/test_native_cpu.py -x -q > gpurun_out/tensor_pytest.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/tensor_pytest.log
