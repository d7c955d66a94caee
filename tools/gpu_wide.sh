#!/bin/bash
# wide secular solver check: tall / cfg4 / hard-case tests, then the 5b timing breakdown
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tall.py tests/test_gpu_parity.py tests/test_gpu_metrics.py tests/test_gpu_acceptance.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_wide.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_wide.log
tail -n 4 gpurun_out/pytest_wide.log
timeout 600 python tools/time_5b.py > gpurun_out/time_5b.log 2>&1; tail -n 15 gpurun_out/time_5b.log
