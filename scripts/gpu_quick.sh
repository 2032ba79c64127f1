#!/bin/bash
# quick iteration: attribution parity tests + C4 ledger timings (linear, step)
timeout 600 python -m pytest tests -x -q -m gpu ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/quick_pytest.log
timeout 300 python scripts/probe_attr.py C4 linear 4 2>&1 | tail -5
timeout 300 python scripts/probe_attr.py C4 step 3 2>&1 | tail -4
