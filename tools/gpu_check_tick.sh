#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/r1_gate_probe.py 99 > gpurun_out/probe_cta.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_vdefer.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ab.log
SHORT="python bench.py --steps 256 --warmup 8 --no-cpu-baseline --e2e-steps 64 --diag-steps 64 --no-k128"
timeout 600 $SHORT > gpurun_out/short.json 2> gpurun_out/short.err
NS="python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 4 --diag-steps 16 --no-k128"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "isvd_timed/" --csv --log-file gpurun_out/launches.csv $NS > gpurun_out/ncu_launch.log 2>&1
FULL="timeout 600 ncu --set full --clock-control none --import-source on"
$FULL -k regex:rank1_fast -s 8 -c 1 -o gpurun_out/r1fast $NS > gpurun_out/ncu_r1fast.log 2>&1
$FULL -k regex:arrow_cta -s 8 -c 1 -o gpurun_out/arrowcta $NS > gpurun_out/ncu_arrowcta.log 2>&1
ls -la gpurun_out | tail -5
