#!/bin/bash
# ncu --set full (with source) of one 5a tick kernel: tools/ncu_one.sh <kernel-regex> <name> [skip]
mkdir -p gpurun_out
SHORT="python bench.py --steps 16 --warmup 3 --no-cpu-baseline --e2e-steps 4 --diag-steps 16 --no-k128"
timeout 300 $SHORT > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$1 -s ${3:-8} -c 1 -o gpurun_out/$2 $SHORT > gpurun_out/ncu_$2.log 2>&1
tail -3 gpurun_out/ncu_$2.log
