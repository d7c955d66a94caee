#!/bin/bash
# rank-1 kernel check: parity / engine tests, short bench, ncu of the new kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py tests/test_gpu_vdefer.py -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_r1.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_r1.log
SHORT="python bench.py --steps 256 --warmup 8 --no-cpu-baseline --e2e-steps 64 --diag-steps 64 --no-k128"
timeout 600 $SHORT > gpurun_out/short.json 2> gpurun_out/short.err || exit 1
NS="python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 4 --diag-steps 16 --no-k128"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rank1_fast -s 8 -c 1 -o gpurun_out/r1fast $NS > gpurun_out/ncu_r1fast.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "isvd_timed/" --csv --log-file gpurun_out/launches.csv $NS > gpurun_out/ncu_launch.log 2>&1
ls -la gpurun_out
