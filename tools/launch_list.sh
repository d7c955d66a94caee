#!/bin/bash
# ncu launch list (gpu__time_duration) of the timed 5a ticks (NVTX range isvd_timed)
mkdir -p gpurun_out
SHORT="python bench.py --steps ${1:-32} --warmup 3 --no-cpu-baseline --e2e-steps 4 --diag-steps 16 --no-k128"
timeout 300 $SHORT > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "isvd_timed/" --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/plain.log | cut -c1-200
