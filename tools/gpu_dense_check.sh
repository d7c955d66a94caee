#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/dense_kernels.py > gpurun_out/dense_kernels.json 2> gpurun_out/dense_kernels.err; cat gpurun_out/dense_kernels.json; tail -3 gpurun_out/dense_kernels.err
timeout 1200 python -m pytest tests/test_gpu_metrics.py tests/test_gpu_tall.py tests/test_gpu_parity.py tests/test_gpu_engine.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_dense.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dense.log; tail -3 gpurun_out/pytest_dense.log
timeout 600 python bench.py --steps 64 --warmup 4 --no-cpu-baseline --e2e-steps 8 --diag-steps 16 --no-k128 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('init_s', d['diagnostics']['init_s'], 'value', d['value'])"
